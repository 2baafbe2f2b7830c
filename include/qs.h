/*
 * qs.h -- C-ABI of the B200-native state-vector hot path of arxiv 2604.12256
 * ("Large-Scale Quantum Circuit Simulation on HPC Cluster via Cache Blocking,
 * Boosting, and Gate Fusion Optimization").
 *
 * Citations: "P:Lx" = /root/reference/PAPER.md line x (section / equation /
 * algorithm named beside it); SURVEY.md 8(b) is the contract these entry
 * points implement.  DESIGN.md lists every reading of the paper (c1..c20).
 *
 * Conventions shared by every call
 *   - Amplitudes are complex128 stored interleaved (re, im): "each state
 *     vector is represented as two 64-bit floating-point numbers"
 *     (Eq. 1).
 *   - Qubit 0 is the least-significant bit of the amplitude index
 *     (reading c1; Eq. 2/3 subscripts P:L129-153).
 *   - A gate matrix over t targets is 2^t x 2^t, row-major; matrix index
 *     bit i <-> targets[i] (reading c2; listing targets ascending gives the
 *     row order of Eq. 3).
 *   - Every call returns QS_OK (0) or a negative QS_E* code; no exception
 *     or signal crosses the ABI.  The message of the last failure on a handle
 *     is available from qs_last_error().
 *   - A handle is not thread-safe; use one handle per thread.
 *   - There is no CPU fallback: a build or machine without a CUDA device
 *     makes qs_create*() fail with QS_ECUDA.
 */
#ifndef QS_H_
#define QS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- errors */
enum {
  QS_OK = 0,
  QS_EINVAL = -1,       /* invalid argument / gate; state left untouched      */
  QS_ENOMEM = -2,       /* device or host allocation failed (bytes in message)*/
  QS_ECUDA = -3,        /* CUDA runtime error; handle is poisoned             */
  QS_ENCCL = -4,        /* NCCL error; handle is poisoned                     */
  QS_EPOISONED = -5,    /* an earlier device failure poisoned the handle      */
  QS_EUNSUPPORTED = -6  /* valid request this build does not implement       */
};

/* ------------------------------------------------------------ gate kinds */
/* SPEC.md L53 kinds + SX/SY/SW (random circuits) + SDG/TDG.  Matrices are
 * reading c3 of DESIGN.md; CX/CZ/CP are X/Z/U1 with >= 1 control. */
enum qs_kind {
  QS_H = 0, QS_X, QS_Y, QS_Z, QS_S, QS_SDG, QS_T, QS_TDG,
  QS_RX, QS_RY, QS_RZ, QS_U1, QS_U2, QS_U3,
  QS_CX, QS_CZ, QS_CP, QS_RZZ, QS_SWAP,
  QS_SX, QS_SY, QS_SW,
  QS_UNITARY,   /* generic 2^t x 2^t unitary given in `matrix`             */
  QS_DIAGONAL,  /* generic diagonal: 2^t unit-modulus entries in `matrix` */
  QS_NUM_KINDS
};

#define QS_MAX_TARGETS 6
#define QS_MAX_CONTROLS 6

/* One gate (`gate`, `targs`).  Controls may name any qubit,
 * including a qubit held on another GPU.  `matrix` (interleaved complex128)
 * is read only for QS_UNITARY (2^t*2^t entries) and QS_DIAGONAL (2^t
 * entries); it is BORROWED for the duration of the call only. */
typedef struct {
  int32_t kind;
  int32_t n_targets;
  int32_t targets[QS_MAX_TARGETS];
  int32_t n_controls;
  int32_t controls[QS_MAX_CONTROLS];
  double params[3];      /* angles in radians: RX/RY/RZ/U1/CP/RZZ: [theta];
                            U2: [phi, lambda]; U3: [theta, phi, lambda]   */
  const double *matrix;
} qs_gate_t;

/* ---------------------------------------------------------------- config */
/* env {N, B, C, R, D, F} of P:L370-374 (Sec. 4.1).  R = log2(#GPUs) is
 * implied by the handle (reading c13). */
#define QS_OPT_BLOCK 1u  /* machine-level cache blocking (Alg. 2) */
#define QS_OPT_FUSE 2u   /* cost-based fusion (GBSA fuse=1)           */
#define QS_OPT_DIAG 4u   /* diagonal detector + fusion (Alg. 8)   */
#define QS_OPT_BOOST 8u  /* merge booster (Alg. 6/7)              */
#define QS_OPT_ALL 15u

typedef struct {
  int32_t chunk_qubits; /* C: chunk = 2^C amplitudes staged per CTA (12)     */
  int32_t fuse_cap;     /* F: max targets of a cost-based fused unitary (4)  */
  int32_t diag_cap;     /* D: max support of a fused diagonal (0 = no cap)   */
  int32_t boost_div;    /* B: Divider(N, ceil(N/B)) (2)                      */
  uint32_t flags;       /* QS_OPT_* (QS_OPT_ALL)                             */
  int32_t jit_min_qubits; /* passes over >= this many local qubits run as
                             per-pass NVRTC-specialised kernels; 0 = all,
                             > 40 = none.  Default 13 (env QS_JIT=0/1
                             overrides the default to none / all).          */
  int32_t l2_block_qubits; /* two-level blocking ("accommodated in
                             the higher-level memory", "within the
                             cache capacity"): consecutive
                             full-state passes whose chunk and output
                             positions all lie below this many qubits run
                             block by block over contiguous blocks of at
                             most 2^this amplitudes, so every pass after
                             the first reads them from L2 instead of
                             HBM (the passes of a run share one
                             cooperative launch, block-level dataflow
                             between them).  0 = off;
                             else 14..40.  Default 0 (measured slower on
                             B200; env QS_L2_BLOCK
                             overrides the default).                      */
} qs_config_t;

/* ----------------------------------------------------------------- stats */
typedef struct {
  uint64_t n_gates_in;       /* gates received by the last qs_apply_circuit   */
  uint64_t n_passes;         /* full-shard passes (chunk + dense + diag)      */
  uint64_t n_chunk_passes, n_dense_passes, n_diag_passes, n_small_passes;
  uint64_t n_expand;         /* booster tensor-product expansions (K5)        */
  uint64_t n_swaps;          /* global<->local exchanges (K4)                 */
  uint64_t n_substate_gates; /* gates simulated on booster sub-states         */
  uint64_t n_fused_diag;     /* fused diagonal groups emitted by Alg. 8       */
  uint64_t bytes_hbm;        /* algorithmic HBM bytes per GPU (32 B/amp/pass) */
  uint64_t bytes_nvlink;     /* bytes sent per GPU by swaps                   */
  uint64_t paper_updates;    /* P:L336/L471 "state vector updates" count      */
  uint64_t naive_updates;    /* G * 2^N                                       */
  double t_plan_ms;          /* host optimiser time of the last call          */
  double t_device_ms;        /* device time of the last call (CUDA events)    */
  double t_swap_ms;          /* part of t_device_ms spent in swaps            */
  uint64_t n_fused_swaps;    /* swaps done by the preceding pass's peer stores
                                 in the last call             */
} qs_stats_t;

typedef struct qs_ctx qs_ctx;

/* ------------------------------------------------------------ lifecycle */
/*
 * qs_create: single process driving `n_gpus` devices (0..n_gpus-1).
 *   n_gpus is a power of two; N_loc = n_qubits - log2(n_gpus) >= 1 and
 *   >= log2(n_gpus); 1 <= n_qubits <= 40.  The state is sharded by its top
 *   log2(n_gpus) physical qubits.  Initial state |0...0>.
 *   Errors: QS_EINVAL, QS_ENOMEM (needed bytes in the message, retrievable
 *   with qs_last_error on the returned handle if *out is non-NULL), QS_ECUDA.
 */
int qs_create(int n_qubits, int n_gpus, qs_ctx **out);

/*
 * qs_create_loopback: `n_ranks` logical ranks whose shards all live on
 * device `device` of this process (exercises the sharded plan and swaps on
 * one GPU; exchanges are device copies).
 */
int qs_create_loopback(int n_qubits, int n_ranks, int device, qs_ctx **out);

/* NCCL unique id (128 bytes) for qs_create_rank; call on rank 0 only and
 * broadcast it (e.g. with torch.distributed). */
int qs_nccl_unique_id(void *id_out_128);

/*
 * qs_create_rank: one process per GPU (torchrun).  Every rank calls it with
 * the same n_qubits/world_size and the same 128-byte NCCL id; this rank
 * owns shard `rank` on CUDA device `device`.  All later calls on the handle
 * are collective (every rank makes the same calls with the same arguments).
 */
int qs_create_rank(int n_qubits, int world_size, int rank, int device,
                   const void *nccl_id_128, qs_ctx **out);

/* qs_destroy: frees every device/host resource of the handle (state shards,
 * receive buffers, descriptor arena, sub-state pool, NCCL communicators,
 * streams, CUDA IPC mappings).  NULL-safe; valid on a poisoned handle.
 * Owns nothing the caller passed in (gate matrices are borrowed per call). */
void qs_destroy(qs_ctx *ctx);

/* ---------------------------------------------------------------- config */
/* qs_set_config: the optimiser environment {C, F, D, B, flags} of Alg. 4
 * (P:L370-374).  chunk_qubits must be 12 (the 2^12-amplitude, 64 KiB chunk
 * of this build); fuse_cap in [1, 4] (4 = one 16x16 register op); diag_cap
 * in [0, 64]; boost_div in [1, 64]; flags within QS_OPT_ALL;
 * jit_min_qubits >= 0.  QS_EINVAL otherwise (config unchanged). */
int qs_set_config(qs_ctx *ctx, const qs_config_t *cfg);
int qs_get_config(const qs_ctx *ctx, qs_config_t *cfg);
/* Defaults: C = 12, F = 4, D = 0 (no cap), B = 2, all flags, jit 18. */
void qs_default_config(qs_config_t *cfg);

/* ----------------------------------------------------------------- state */
/* |x> (x < 2^n).  Marks the state as a known product state, which enables
 * the merge booster for the next qs_apply_circuit (reading c10).  No device
 * work happens until the state is used. */
int qs_set_basis_state(qs_ctx *ctx, uint64_t x);

/*
 * qs_apply_circuit: optimise (Alg. 4 swarm optimisation) and
 * apply `n_gates` gates in order (the result is that of Alg. 1).
 * Synchronous.  Validation happens before any device work; on QS_EINVAL the
 * state is untouched: index >= N, duplicate/overlapping targets/controls,
 * t > 6, ||U U^+ - I||_inf >= 1e-10, |lambda| != 1 +- 1e-10 (SPEC.md
 * L55-57).  A CUDA/NCCL failure returns QS_ECUDA/QS_ENCCL and poisons the
 * handle (state undefined; only qs_destroy is valid).
 */
int qs_apply_circuit(qs_ctx *ctx, const qs_gate_t *gates, size_t n_gates);

/*
 * qs_get_state: amplitudes alpha_i, i in [offset, offset+count), of the state
 * vector |psi> = sum_i alpha_i |i> of Eq. 1 ("two 64-bit
 * floating-point numbers" each) in LOGICAL index order: qubit q is bit q of
 * i (reading c1); the virtual qubit map (Eq. 4 reordering) and
 * the sharding by the top log2(P) qubits are undone on the device (K6).
 * host_out: caller-owned host buffer of 2*count doubles (re, im interleaved;
 * pinned memory makes it one DMA).  Collective in rank mode (every rank
 * receives the slice).  Errors: QS_EINVAL (NULL buffer with count > 0,
 * range beyond 2^n), QS_EPOISONED, QS_ECUDA/QS_ENCCL (handle poisoned).
 */
int qs_get_state(qs_ctx *ctx, double *host_out, uint64_t offset, uint64_t count);

/*
 * qs_probabilities: |alpha_i|^2 (Eq. 1: the measurement
 * probability of basis state |i>) for the same logical slice into the
 * caller-owned host buffer `host_out` of count doubles.  Same ordering,
 * collectivity and errors as qs_get_state.
 */
int qs_probabilities(qs_ctx *ctx, double *host_out, uint64_t offset, uint64_t count);

/* qs_get_stats: plan and timing statistics of the last qs_apply_circuit
 * (qs_stats_t above; paper_updates = the "state vector updates" count of
 * P:L336/L471, t_plan_ms = the optimiser time P:L382 bounds).  QS_EINVAL on
 * NULL arguments. */
int qs_get_stats(const qs_ctx *ctx, qs_stats_t *out);
/* Message of the last failure on the handle (owned by the handle, valid until
 * the next call on it); "NULL handle" for NULL. */
const char *qs_last_error(const qs_ctx *ctx);

/* ---------------------------------------------------- plan inspection (host) */
/*
 * Host-only planning, no device needed: runs the same optimiser as
 * qs_apply_circuit for an n_qubits state sharded over n_ranks and writes a
 * JSON description of the plan (steps, passes, phases, swaps, statistics)
 * into `buf` (NUL-terminated, truncated to `cap`).  Returns the length the
 * full text needs (excluding the NUL), or a negative QS_E* code (then `buf`
 * holds the error message).
 * `product_state` != 0 plans from the basis state |basis> (booster allowed).
 * `detail` != 0 adds every op's matrix / phase monomials (64-bit values as
 * decimal strings) so a test can replay the plan.
 */
int64_t qs_plan_json(int n_qubits, int n_ranks, const qs_config_t *cfg,
                     int product_state, uint64_t basis,
                     const qs_gate_t *gates, size_t n_gates, int detail,
                     char *buf, size_t cap);

/* Alg. 6 Divider(N, divSize): writes the group sizes into
 * out[] (capacity cap); returns the number of groups or a QS_E* code. */
int qs_divider(int n, int div_size, int *out, int cap);

/* ------------------------------------------------------------ diagnostics */
/* Number of kernel launches this handle issued during the last
 * qs_apply_circuit (all ranks' shards owned by this process). */
uint64_t qs_last_launches(const qs_ctx *ctx);

/* Per-kernel device timing of the last qs_apply_circuit (CUDA events
 * recorded around every launch on the launching stream of the first local
 * shard).  Enabled by default; qs_set_timing(ctx, 0) disables it;
 * qs_set_timing(ctx, 2) makes the per-kernel timings, qs_last_launches and
 * the t_plan_ms / t_device_ms statistics ADD UP over the following calls
 * (a benchmark reads them once after its timed loop).  Every call of
 * qs_set_timing resets them. */
enum qs_kernel_id {
  QS_K1_CHUNK = 0,  /* multi-layout chunk kernel                          */
  QS_K2_DENSE = 1,  /* single-layout dense (fused matvec) pass            */
  QS_K3_DIAG = 2,   /* diagonal phase pass                                */
  QS_K_SMALL = 3,   /* whole-shard kernel for <= 2^12 amplitudes          */
  QS_K5_EXPAND = 4, /* booster tensor-product expansion                   */
  QS_K5_MERGE = 5,  /* booster sub-state merge                            */
  QS_K_INIT = 6,    /* basis-state initialisation                         */
  QS_K4_SWAP = 7,   /* global<->local exchange                            */
  QS_K6_READ = 8,
  QS_K_SUBSTATE = 9, /* any pass on a booster sub-state (K1/K2/K3/SMALL)  */
  QS_K1_FUSED_SWAP = 10, /* full-state pass that also performs the following
                            swap's exchange by NVLink peer stores (f1):
                            its time covers the pass AND the transfer       */
  QS_K1_PULL = 11,       /* the pass after a split fused swap: it loads the
                            half the exporting pass left in place from the
                            source ranks' buffers (NVLink reads)            */
  QS_K1_L2_GROUP = 12    /* a run of passes executed wave by wave over
                            L2-sized blocks (two-level blocking, f2): one
                            entry per run; bytes = the run's HBM bytes      */
};
int qs_set_timing(qs_ctx *ctx, int enable);
/* The cudaStream_t (as void*) the handle launches local shard `i` on, so a
 * caller can record its own CUDA events on the launching stream; NULL if
 * out of range.  Owned by the handle. */
void *qs_get_stream(const qs_ctx *ctx, int i);

/* Pass specialisation (NVRTC, sm_100a): the chunk/dense/diagonal passes of
 * large shards are compiled per pass structure and cached (QS_JIT=0|1|auto;
 * cache directory QS_JIT_CACHE; all passes of a call are prepared -- in
 * parallel -- before its first launch).  Writes a JSON object {jit_launches,
 * jit_errors, compile_ms, compiles, disk_hits, prep_ms, variants:
 * {write_only, bulk_tma, tensor_tma, cp_async}, last_error} (process-wide
 * compile counters; launch counters of this handle, per chunk refill engine;
 * prep_ms = kernel preparation time of the last call) into buf; returns its
 * length. */
int64_t qs_jit_info(const qs_ctx *ctx, char *buf, size_t cap);
/* launches, summed device ms and ALGORITHMIC bytes (32 B per amplitude per
 * read+write pass, 16 B for write-only passes; swap: bytes sent). */
int qs_get_kernel_timing(const qs_ctx *ctx, int kernel_id, uint64_t *launches,
                         double *ms, uint64_t *bytes);

#ifdef __cplusplus
}
#endif
#endif /* QS_H_ */
