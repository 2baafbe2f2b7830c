// qs_internal.hpp -- internal types of libqs (host planner <-> executor <->
// kernels).  Not part of the ABI; see include/qs.h for the boundary.
//
// The device "pass descriptor" (KPass*) is a flat POD blob produced by the
// host planner (planner.cpp) and consumed by the kernels (kernels.cu).
#pragma once
#include <stdint.h>

#include <string>

namespace qs {

typedef uint64_t u64;

// ---------------------------------------------------------------- geometry
constexpr int kRegBits = 4;               // register-resident qubits / thread
constexpr int kNReg = 1 << kRegBits;      // 16 amplitudes per thread
constexpr int kLogT = 8;                  // 256 threads per CTA
constexpr int kThreads = 1 << kLogT;
constexpr int kChunkBits = kLogT + kRegBits;  // m = 12 -> 4096 amps = 64 KiB
constexpr int kSmallMax = 12;             // shards with nl <= 12 -> SMALL kernel
constexpr int kMaxPhases = 8;             // register layouts per chunk pass
constexpr int kMaxShapes = 1024;          // diag shapes per pass (smem)
constexpr int kMaxRuns = 16;              // runs of the chunk-id deposit
constexpr int kMaxExpand = 4;             // sub-states multiplied by K5
constexpr int kMaxVaryTab = 64;           // chunk-dependent shapes read from a table
constexpr int kMaxRun = 4;                 // passes per co-scheduled run (f2)
constexpr int kMaxXBits = 3;              // fused-swap export bits (2^3 destinations)

// Kernel kinds (stats / timing ids).
enum KernelKind {
  KK_CHUNK = 0,   // K1: multi-phase chunk kernel (smem exchanges)
  KK_DENSE = 1,   // K2: single-phase dense pass (registers only)
  KK_DIAG = 2,    // K3: single-phase diagonal pass
  KK_SMALL = 3,   // whole shard in one CTA (nl <= 12)
  KK_EXPAND = 4,  // K5 standalone tensor-product expansion
  KK_MERGE = 5,   // K5 sub-state merge
  KK_INIT = 6,    // basis-state initialisation
  KK_SWAP = 7,    // K4 exchange (NCCL / copies)
  KK_READ = 8,    // K6 readout gather
  KK_SUB = 9,     // passes on booster sub-states (timing class only)
  KK_XPASS = 10,  // full-state pass that also performs the next swap's
                  // exchange by NVLink peer stores (f1; timing class only)
  KK_PULL = 11,   // full-state pass that loads the other half of a split
                  // swap from the source ranks' buffers (timing class only)
  KK_L2 = 12,     // a run of passes executed wave by wave over L2-sized
                  // blocks (f2; timing class only)
  KK_NUM = 13
};

// Register-op types inside a pass.
enum OpType : uint8_t {
  OP_D1 = 1,    // dense 2x2 on register bit `sel`
  OP_D2 = 2,    // dense 4x4 on register-bit pair `sel` (pair code)
  OP_D3 = 3,    // dense 8x8 on register bits {0..3} \ {sel}
  // (4: unused -- 4-target ops run as OP_DW: a 16x16 in registers needs
  //  16 inputs + 16 outputs live, all 128 registers of a thread)
  OP_H = 5,     // Hadamard on register bit `sel`
  OP_X = 6,     // Pauli X on register bit `sel` (register swap)
  OP_DIAG = 7,  // phase polynomial group `data`, general path (2^a sincos)
  OP_DIAGF = 8, // fast path: sincos only for the varying empty/linear
                // register subsets (sel = linear mask L), register-pair
                // terms constant (host table CK16), rcm = touched-rho mask
  OP_HU = 9,    // unnormalised Hadamard (x+y, x-y); pass scale at the store
  OP_DW = 10,   // wide dense 2^k x 2^k (k = 4..6) applied to the chunk in
                // shared memory at the exchange into its layout: k targets =
                // chunk bits tpos[0..k), chunk-bit control mask rcm, physical
                // non-chunk control mask ncm, matrix at pool offset data
                // (row-major, matrix bit i <-> tpos[i]); first op of a layout
  // SMALL kernel ops (physical positions, whole shard in smem)
  OP_SDENSE = 20,
  OP_SDIAG = 21,
};

// Pair code for OP_D2: index into {(0,1),(0,2),(0,3),(1,2),(1,3),(2,3)}.

struct KOp {
  uint8_t type;
  uint8_t sel;       // register bit / pair code / missing bit / active mask
  uint8_t k;         // number of targets (SMALL ops)
  uint8_t has_const; // OP_DIAG: some shape has an empty register part
  uint32_t rcm;      // control mask over the register index rho
  u64 ncm;           // physical control mask of non-register bits (incl. rank)
  int32_t data;      // pool offset (doubles) of the matrix, or group index
  int32_t data2;     // SMALL OP_SDIAG: term count
  int8_t tpos[8];    // SMALL: physical target positions (matrix bit i)
};

struct KPhase {
  int8_t reg_c[kRegBits];   // chunk bit of register bit k
  int8_t thr_c[10];         // chunk bit of tid bit i
  int16_t op_begin, op_end;
};

// One diagonal group evaluated in one phase: shapes sorted by their register
// subset R, rbeg[R]..rbeg[R+1].
struct KGroup {
  int32_t rbeg[17];
  int32_t ck_off;   // OP_DIAGF: pool offset (doubles) of CK16[16], -1 if none
};

// A "shape": monomials that agree on their chunk bits.  Its coefficient is
// computed once per chunk (level 1) from its terms; a thread adds it when its
// thread bits cover `tmask` (level 2).
struct KShape {
  uint32_t tmask;      // mask over tid bits (phase layout)
  int32_t term_begin;
  int32_t term_end;
  int32_t pad;
};

struct KTerm {
  u64 ncmask;   // physical mask of the non-chunk bits (incl. rank bits)
  u64 coeff;    // angle in turns * 2^64 (mod 2^64)
};

struct KExpand {
  u64 ptr[kMaxExpand];      // device pointers (double2*) of sub-states
  int32_t lo[kMaxExpand];   // lowest physical bit of the group
  int32_t len[kMaxExpand];  // group width
  int32_t n;
  int32_t pad;
};

struct KPass {
  int32_t kernel;      // KernelKind
  int32_t nl;          // local qubits of the target buffer
  int32_t n_phases;
  int32_t n_ops;
  int32_t n_shapes;
  int32_t n_runs;
  int32_t src_mode;    // 0 load; 1 phase-0 amplitudes from `expand`; 2 basis
  int32_t n_groups;
  u64 n_chunks;
  u64 rank_base;       // rank << nl
  u64 local_mask;      // (1 << nl) - 1
  u64 basis;           // src_mode 2: physical index of the 1.0 amplitude
  double scale;        // (scale, scale_im) multiplies every amplitude: the
  double scale_im;     // 2^{-1/2} of each OP_HU and the scalars factored out
                       // of unit-scaled dense ops (encode_pass)
  int32_t x_shift, x_mask;  // fused swap export: x_mask = 2^j - 1 (0: none)
  int8_t x_pos[8];          // piece s = sum_i bit x_pos[i] of the local index << i
  int8_t x_split;           // push only chunks whose bit x_split is 0 (-1: all)
  int8_t pull_j, pull_z;    // pull pass: source table entry (z << 3) | piece
  int8_t pull_pos[5];       //   piece = sum_i bit pull_pos[i] << i
  int8_t cpos[16];     // physical position of chunk bit c (loads, ops)
  int8_t opos[16];     // physical position of chunk bit c (stores; relabel)
  int8_t run_src[kMaxRuns], run_dst[kMaxRuns], run_len[kMaxRuns];
  KPhase phases[kMaxPhases];
  KExpand expand;
  uint32_t off_ops, off_groups, off_shapes, off_terms, off_pool;
  uint32_t total_bytes;
};

// Per-chunk table of a specialised pass (qs_kshape_table), one row per chunk:
//  - angle columns: the level-1 sum of a chunk-dependent shape (u64 turns);
//  - cis columns: exp(2 pi i sum/2^64) of the summed shapes of one diagonal
//    slot whose chunk-dependent part does not depend on the thread (a
//    double2, so the pass takes no sincos for it).
// Row = n_ang angles, padded to even, then 2 u64 per cis column.
constexpr int kMaxTabCis = 32;
constexpr int kMaxTabRefs = 192;
struct TabCols {
  int32_t n_ang, n_cis;
  int16_t ang[kMaxVaryTab];
  int16_t cis_beg[kMaxTabCis + 1];
  int16_t cis_shape[kMaxTabRefs];
  int32_t width;  // u64 per row: ((n_ang + 1) & ~1) + 2 * n_cis
};

// Refill engine of a specialised pass (qs_jit_info counts launches per kind).
enum JitVariant {
  JV_WRITE_ONLY = 0,  // source fused (booster expand / basis): no loads
  JV_BULK = 1,        // cp.async.bulk (TMA bulk copies) of >= 512 B runs
  JV_TENSOR = 2,      // one cp.async.bulk.tensor per chunk
  JV_CPASYNC = 3,     // per-thread cp.async (128-256 B runs)
  JV_NUM = 4
};

// A specialised kernel ready to launch (or why not).
struct JitPrepared {
  bool ok = false;
  void* fn = nullptr;   // CUfunction
  int per_sm = 1;       // resident CTAs per SM
  int threads = kThreads;
  size_t smem = 0;
  int variant = 0;      // JitVariant
  int grid_mult = 1;    // launch grid must be a multiple of this
  std::string err;
};

}  // namespace qs
