// api.cpp -- C-ABI entry points (include/qs.h) and the plan executor.
//
// One handle owns one or more shards (a shard = 2^nl amplitudes of the
// state, rank r holds physical indices [r*2^nl, (r+1)*2^nl)).
// Three ownership modes:
//   single   qs_create(n, P): this process drives devices 0..P-1 (NCCL comms
//            from ncclCommInitAll; exchanges over NVLink);
//   loopback qs_create_loopback(n, P, dev): P shards on one device, the
//            exchange is device copies (CI for the sharded path on one GPU);
//   rank     qs_create_rank(...): one process per GPU (torchrun), NCCL comm
//            from a broadcast unique id.
// Every step of the hot path runs in the kernels of kernels.cu or in NCCL;
// there is no host compute fallback.
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/qs.h"
#include "planner.hpp"
#include "qs_internal.hpp"

namespace qs {
cudaError_t launch_pass(int kernel, const unsigned char* dblob, const KPass& hdr,
                        double2* state, cudaStream_t st);
cudaError_t launch_expand(double2* dst, u64 n_amps, u64 rank_base, const KExpand& e,
                          cudaStream_t st);
cudaError_t launch_merge(double2* dst, const double2* A, int la, const double2* B, int lb,
                         cudaStream_t st);
cudaError_t launch_set_one(double2* dst, u64 idx, cudaStream_t st);
cudaError_t launch_permute(const double2* in, double2* out, u64 n_amps, const int* a, const int* b,
                           int n, cudaStream_t st);
cudaError_t launch_gather(const double2* state, double2* out, u64 off, u64 count, int n,
                          const int8_t* dmap, int nl, u64 rank, int probs, cudaStream_t st);
bool jit_prepare(const unsigned char* blob, int device, void** fn_out, int* grid_per_sm,
                 size_t* smem_out, std::string& err, bool compile_only);
int jit_prepare_all(const std::vector<const unsigned char*>& blobs, int device,
                    std::vector<JitPrepared>& out, bool compile_only);
cudaError_t jit_launch(void* fn, int grid, size_t smem, const unsigned char* dblob,
                       const unsigned char* hblob, double2* state, u64 rank_base, const u64* vtab,
                       const u64* xpeer8, const void* pool_host, size_t pool_bytes, cudaStream_t st,
                       u64 clo, u64 cn);
int jit_table_cols(const unsigned char* blob, TabCols* v);
bool jit_prepare_run(const std::vector<const unsigned char*>& blobs, int sb, int device, JitPrepared& out,
                     bool compile_only = false);
cudaError_t jit_launch_run(const JitPrepared& jp, int grid, const std::vector<const unsigned char*>& dblobs,
                           const std::vector<const unsigned char*>& hblobs, double2* state, u64 rank_base,
                           const std::vector<const u64*>& vtabs, u64 n_chunks, unsigned* flags, unsigned nblk,
                           const unsigned* split, unsigned lag, cudaStream_t st);
cudaError_t launch_shape_table(const unsigned char* dblob, u64* tab, u64 rank_base, u64 n_chunks,
                               const TabCols& v, cudaStream_t st);
size_t jit_param_bytes(const unsigned char* blob);
void jit_stats(double* compile_ms, uint64_t* compiles, uint64_t* disk_hits);
}  // namespace qs

namespace {
// QS_JIT: "0" interpreter kernels only, "1" specialise every chunk/dense/diag
// pass, unset/"auto": specialise every pass over more than kSmallMax local
// qubits, booster sub-states included (round 2: the 15-qubit sub-state
// passes of QFT-30 on the interpreter cost ~0.1 ms per circuit, 8.93 ->
// 8.84 ms; the others tie; round 1 kept them on the interpreter, 18).
int jit_default_min() {
  const char* e = getenv("QS_JIT");
  if (!e || !*e || !strcmp(e, "auto")) return qs::kSmallMax + 1;
  return atoi(e) ? 0 : 99;
}

int num_sms_of(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cache[device] = v > 0 ? v : 148;
  }
  return cache[device];
}
}  // namespace

using namespace qs;

namespace {

enum Mode { M_SINGLE = 0, M_LOOPBACK = 1, M_RANK = 2 };

struct Timed {
  int kind;
  cudaEvent_t a, b;
  uint64_t bytes;
};

struct Shard {
  int device = 0;
  int rank = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double2* state = nullptr;
  double2* scratch = nullptr;        // swap receive buffer
  ncclComm_t comm = nullptr;
  unsigned char* arena = nullptr;    // pass descriptors (device)
  size_t arena_cap = 0;
  double2* subpool = nullptr;        // booster sub-states (device)
  size_t subpool_cap = 0;            // amplitudes
  double2* tmp = nullptr;            // readout gather buffer
  size_t tmp_cap = 0;                // amplitudes
  int8_t* dmap = nullptr;            // logical->physical map (device)
  unsigned* l2flags = nullptr;       // per-block counters of co-scheduled runs (f2)
  size_t l2flags_cap = 0;            // bytes
  u64* vtab = nullptr;               // per-chunk shape sums of the running pass
  size_t vtab_cap = 0;               // entries
  cudaStream_t side = nullptr;       // per-chunk tables of all passes, computed
                                     // ahead of their passes (overlapping them)
  double2* alloc[2] = {nullptr, nullptr};  // the two shard allocations (state,
                                           // scratch at creation; they alternate)
  double* bar = nullptr;             // rank mode: 1-element all-reduce = barrier
  std::vector<Timed> timed;          // per-launch events of the last call
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
};

}  // namespace

struct qs_ctx {
  int n = 0, n_ranks = 1, n_global = 0, nl = 0;
  Mode mode = M_SINGLE;
  std::vector<Shard> shards;
  qs_config_t cfg;
  std::vector<int> map;              // logical -> physical
  bool pending = true;               // state not yet written: it is |basis>
  uint64_t basis = 0;
  bool poisoned = false;
  std::string err;
  qs_stats_t stats;
  uint64_t launches = 0;
  unsigned char* host_stage = nullptr;  // pinned staging for descriptors
  size_t host_stage_cap = 0;
  double* host_tmp = nullptr;           // pinned readout staging
  size_t host_tmp_cap = 0;
  bool timing = true;
  bool accumulate = false;  // qs_set_timing(ctx, 2): timings/launches/plan and device
                            // times add up over calls until the next qs_set_timing
  uint64_t jit_launches = 0, jit_errors = 0;
  uint64_t n_l2_groups = 0;               // runs executed wave by wave (f2)
  uint64_t jit_variant[JV_NUM] = {0, 0, 0, 0};  // launches per refill engine (handle lifetime)
  double prep_ms = 0;                           // last call: kernel preparation (compile/load)
  std::string jit_last_error;
  // fused swaps: pointer swaps so far (all shards and ranks
  // in lockstep), peer access state (0 unknown, 1 ready, -1 unavailable),
  // rank mode: the peers' two allocations mapped through CUDA IPC
  uint64_t swap_parity = 0;
  int peers = 0;
  std::vector<double2*> ipc;
  bool fused_pending = false;
  // the last circuit's launches are enqueued but not yet waited for
  // (accumulating timing mode: finish_inflight)
  bool inflight = false;
  uint64_t n_fused_swaps = 0;
  // per kernel kind: launches, ms, algorithmic bytes (last call, shard 0..)
  uint64_t k_count[KK_NUM];
  double k_ms[KK_NUM];
  uint64_t k_bytes[KK_NUM];
};

namespace {

int set_err(qs_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CU(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      ctx->poisoned = true;                                                       \
      return set_err(ctx, QS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                             \
  } while (0)

#define NC(call)                                                                  \
  do {                                                                            \
    ncclResult_t r_ = (call);                                                     \
    if (r_ != ncclSuccess) {                                                      \
      ctx->poisoned = true;                                                       \
      return set_err(ctx, QS_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    }                                                                             \
  } while (0)

int log2i(int x) {
  int l = 0;
  while ((1 << l) < x) l++;
  return ((1 << l) == x) ? l : -1;
}

cudaEvent_t get_event(Shard& s) {
  if (s.ev_used == s.ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    s.ev_pool.push_back(e);
  }
  return s.ev_pool[s.ev_used++];
}

int alloc_shard_memory(qs_ctx* ctx, Shard& s) {
  CU(cudaSetDevice(s.device));
  const size_t bytes = (size_t)16 << ctx->nl;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  size_t need = bytes * ((ctx->n_ranks > 1) ? 2 : 1);
  if (ctx->mode == M_LOOPBACK) need = 0;  // checked once by the caller
  if (need > fr) {
    char b[200];
    snprintf(b, sizeof b, "need %zu bytes on device %d, %zu free", need, s.device, fr);
    return set_err(ctx, QS_ENOMEM, b);
  }
  if (cudaMalloc(&s.state, bytes) != cudaSuccess)
    return set_err(ctx, QS_ENOMEM, "cudaMalloc state failed (" + std::to_string(bytes) + " B)");
  if (ctx->n_ranks > 1 && cudaMalloc(&s.scratch, bytes) != cudaSuccess)
    return set_err(ctx, QS_ENOMEM, "cudaMalloc swap buffer failed (" + std::to_string(bytes) + " B)");
  CU(cudaMalloc(&s.dmap, 64));
  s.alloc[0] = s.state;
  s.alloc[1] = s.scratch;
  if (ctx->n_ranks > 1) {
    CU(cudaMalloc(&s.bar, 64));
    CU(cudaMemset(s.bar, 0, 64));
  }
  CU(cudaEventCreate(&s.t0));
  CU(cudaEventCreate(&s.t1));
  return QS_OK;
}

void init_ctx(qs_ctx* ctx, int n, int n_ranks) {
  ctx->n = n;
  ctx->n_ranks = n_ranks;
  ctx->n_global = log2i(n_ranks);
  ctx->nl = n - ctx->n_global;
  qs_default_config(&ctx->cfg);
  ctx->map.resize(n);
  for (int q = 0; q < n; q++) ctx->map[q] = q;
  ctx->pending = true;
  ctx->basis = 0;
  memset(&ctx->stats, 0, sizeof ctx->stats);
  memset(ctx->k_count, 0, sizeof ctx->k_count);
  memset(ctx->k_ms, 0, sizeof ctx->k_ms);
  memset(ctx->k_bytes, 0, sizeof ctx->k_bytes);
}

int check_dims(int n, int n_ranks, std::string& why) {
  if (n < 1 || n > 40) { why = "n_qubits must be in [1, 40]"; return QS_EINVAL; }
  const int g = log2i(n_ranks);
  if (n_ranks < 1 || g < 0) { why = "rank count must be a power of two"; return QS_EINVAL; }
  const int nl = n - g;
  if (nl < 1 || nl < g) { why = "too few local qubits for this rank count"; return QS_EINVAL; }
  return QS_OK;
}

int ensure_host_stage(qs_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->host_stage_cap) return QS_OK;
  if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
  size_t cap = std::max(bytes, (size_t)1 << 20);
  CU(cudaMallocHost(&ctx->host_stage, cap));
  ctx->host_stage_cap = cap;
  return QS_OK;
}

// ------------------------------------------------------------ fused swap
// a pass right before a swap stores the pieces it exports
// straight into the receive buffers of their destination ranks (NVLink peer
// stores), so the exchange overlaps the pass instead of following it.  Needs
// every receive buffer addressable: same device (loopback), peer access
// (one process, several GPUs), or CUDA IPC mappings (one process per GPU;
// handles exchanged once over the NCCL communicator).
int ensure_peers(qs_ctx* ctx) {
  if (ctx->peers) return ctx->peers;
  ctx->peers = -1;
  if (getenv("QS_NO_FUSED_SWAP") || ctx->n_ranks < 2) return ctx->peers;
  if (ctx->mode == M_LOOPBACK) {
    ctx->peers = 1;
  } else if (ctx->mode == M_SINGLE) {
    for (Shard& a : ctx->shards)
      for (Shard& b : ctx->shards) {
        if (a.device == b.device) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, a.device, b.device);
        if (!can) return ctx->peers;
        cudaSetDevice(a.device);
        cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return ctx->peers;
      }
    ctx->peers = 1;
  } else {
    // every rank takes part in both collectives (handle all-gather, then a
    // min-vote on success) so that all of them make the same decision
    Shard& sh = ctx->shards[0];
    cudaSetDevice(sh.device);
    cudaIpcMemHandle_t h[2];
    memset(h, 0, sizeof h);
    bool ok = cudaIpcGetMemHandle(&h[0], sh.alloc[0]) == cudaSuccess &&
              cudaIpcGetMemHandle(&h[1], sh.alloc[1]) == cudaSuccess;
    if (!ok) cudaGetLastError();
    const size_t hb = sizeof h;
    unsigned char* d = nullptr;
    if (cudaMalloc(&d, hb * ctx->n_ranks + 16) != cudaSuccess) return ctx->peers;
    std::vector<unsigned char> all(hb * ctx->n_ranks);
    bool coll = cudaMemcpyAsync(d + hb * sh.rank, h, hb, cudaMemcpyHostToDevice, sh.stream) == cudaSuccess &&
                ncclAllGather(d + hb * sh.rank, d, hb, ncclUint8, sh.comm, sh.stream) == ncclSuccess &&
                cudaMemcpyAsync(all.data(), d, all.size(), cudaMemcpyDeviceToHost, sh.stream) == cudaSuccess &&
                cudaStreamSynchronize(sh.stream) == cudaSuccess;
    ok = ok && coll;
    std::vector<double2*> mapped(2 * ctx->n_ranks, nullptr);
    for (int r = 0; r < ctx->n_ranks && ok; r++) {
      if (r == sh.rank) {
        mapped[2 * r] = sh.alloc[0];
        mapped[2 * r + 1] = sh.alloc[1];
        continue;
      }
      for (int k = 0; k < 2 && ok; k++) {
        cudaIpcMemHandle_t hk;
        memcpy(&hk, all.data() + hb * r + sizeof(cudaIpcMemHandle_t) * k, sizeof hk);
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, hk, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          ok = false;
        } else {
          mapped[2 * r + k] = (double2*)p;
        }
      }
    }
    double vote = ok ? 1.0 : 0.0;
    double* dv = reinterpret_cast<double*>(d + hb * ctx->n_ranks);
    coll = coll && cudaMemcpyAsync(dv, &vote, sizeof vote, cudaMemcpyHostToDevice, sh.stream) == cudaSuccess &&
           ncclAllReduce(dv, dv, 1, ncclDouble, ncclMin, sh.comm, sh.stream) == ncclSuccess &&
           cudaMemcpyAsync(&vote, dv, sizeof vote, cudaMemcpyDeviceToHost, sh.stream) == cudaSuccess &&
           cudaStreamSynchronize(sh.stream) == cudaSuccess;
    cudaFree(d);
    ctx->ipc = mapped;  // closed at destroy (whatever was opened)
    if (coll && vote == 1.0) ctx->peers = 1;
  }
  return ctx->peers;
}

// Receive buffer of rank d right now (the two allocations alternate with
// every pointer swap, in lockstep on all ranks).
double2* recv_buffer(qs_ctx* ctx, int d) {
  if (ctx->mode != M_RANK) return ctx->shards[d].scratch;
  return ctx->ipc[2 * d + ((ctx->swap_parity & 1) ? 0 : 1)];
}

// Destination bases of rank r's exported pieces for the swap `st`: local
// index i whose bits at lpos spell s goes to rank dest(r, s), at i with
// those bits replaced by u(r) -- so the base is that rank's receive buffer
// + (dep(u(r)) - dep(s)) amplitudes, dep(v) placing bit i of v at lpos[i].
void fused_targets(qs_ctx* ctx, const Step& st, int r, u64 out[1 << kMaxXBits]) {
  const int j = st.j, nl = ctx->nl;
  auto dep = [&](int v) {
    u64 x = 0;
    for (int i = 0; i < j; i++) x |= (u64)((v >> i) & 1) << st.lpos[i];
    return x;
  };
  int ur = 0;
  for (int i = 0; i < j; i++) ur |= ((r >> (st.gpos[i] - nl)) & 1) << i;
  for (int s = 0; s < (1 << kMaxXBits); s++) {
    out[s] = 0;
    if (s >= (1 << j)) continue;
    int d = r;
    for (int i = 0; i < j; i++) d = (d & ~(1 << (st.gpos[i] - nl))) | (((s >> i) & 1) << (st.gpos[i] - nl));
    out[s] = (u64)recv_buffer(ctx, d) + (dep(ur) - dep(s)) * sizeof(double2);
  }
}

// Device-side barrier over every shard's stream (rank mode: a 1-element
// NCCL all-reduce; in-process: each stream waits for the others' events).
int shard_barrier(qs_ctx* ctx) {
  if (ctx->mode == M_RANK) {
    for (Shard& sh : ctx->shards) {
      CU(cudaSetDevice(sh.device));
      NC(ncclAllReduce(sh.bar, sh.bar, 1, ncclDouble, ncclSum, sh.comm, sh.stream));
    }
    return QS_OK;
  }
  if (ctx->shards.size() < 2) return QS_OK;
  std::vector<cudaEvent_t> done;
  for (Shard& sh : ctx->shards) {
    CU(cudaSetDevice(sh.device));
    done.push_back(get_event(sh));
    CU(cudaEventRecord(done.back(), sh.stream));
  }
  for (size_t t = 0; t < ctx->shards.size(); t++) {
    CU(cudaSetDevice(ctx->shards[t].device));
    for (size_t u = 0; u < done.size(); u++)
      if (u != t) CU(cudaStreamWaitEvent(ctx->shards[t].stream, done[u], 0));
  }
  return QS_OK;
}

bool top_lpos(const qs_ctx* ctx, const Step& st) {
  for (int i = 0; i < st.j; i++)
    if (st.lpos[i] != ctx->nl - st.j + i) return false;
  return true;
}

// ----------------------------------------------------------------- swap
// Exchange global positions gpos[i] with local positions lpos[i] = nl-j+i.
// Piece s (top j local bits) of rank r goes to rank r with bits b_i := s_i,
// landing at its piece u(r) (a pure relabel afterwards).
int exec_swap(qs_ctx* ctx, const Step& st) {
  const int j = st.j, nl = ctx->nl;
  const size_t piece = (size_t)1 << (nl - j);          // amplitudes
  const size_t pbytes = piece * sizeof(double2);
  std::vector<int> b(j);
  for (int i = 0; i < j; i++) b[i] = st.gpos[i] - nl;
  auto u_of = [&](int r) {
    int u = 0;
    for (int i = 0; i < j; i++) u |= ((r >> b[i]) & 1) << i;
    return u;
  };
  auto dest = [&](int r, int s) {
    int d = r;
    for (int i = 0; i < j; i++) d = (d & ~(1 << b[i])) | (((s >> i) & 1) << b[i]);
    return d;
  };
  if (ctx->mode == M_LOOPBACK) {
    Shard& s0 = ctx->shards[0];
    CU(cudaSetDevice(s0.device));
    for (Shard& sh : ctx->shards) {
      const int r = sh.rank, ur = u_of(r);
      for (int s = 0; s < (1 << j); s++) {
        Shard& dst = ctx->shards[dest(r, s)];
        CU(cudaMemcpyAsync(dst.scratch + (size_t)ur * piece, sh.state + (size_t)s * piece,
                           pbytes, cudaMemcpyDeviceToDevice, s0.stream));
      }
    }
  } else {
    NC(ncclGroupStart());
    for (Shard& sh : ctx->shards) {
      const int r = sh.rank, ur = u_of(r);
      for (int s = 0; s < (1 << j); s++) {
        if (s == ur) continue;
        const int d = dest(r, s);
        NC(ncclSend(sh.state + (size_t)s * piece, 2 * piece, ncclDouble, d, sh.comm, sh.stream));
        NC(ncclRecv(sh.scratch + (size_t)s * piece, 2 * piece, ncclDouble, d, sh.comm, sh.stream));
      }
    }
    NC(ncclGroupEnd());
    for (Shard& sh : ctx->shards) {
      CU(cudaSetDevice(sh.device));
      const int ur = u_of(sh.rank);
      CU(cudaMemcpyAsync(sh.scratch + (size_t)ur * piece, sh.state + (size_t)ur * piece, pbytes,
                         cudaMemcpyDeviceToDevice, sh.stream));
    }
  }
  for (Shard& sh : ctx->shards) std::swap(sh.state, sh.scratch);
  return QS_OK;
}

// -------------------------------------------------------------- execute
int execute_steps(qs_ctx* ctx, const Plan& plan);
int finish_inflight(qs_ctx* ctx);

// Every error after the first launch leaves a partly applied circuit:
// the handle is poisoned (include/qs.h, qs_apply_circuit).
int execute(qs_ctx* ctx, const Plan& plan) {
  const int rc = execute_steps(ctx, plan);
  if (rc && ctx->launches) ctx->poisoned = true;
  return rc;
}

static double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

int execute_steps(qs_ctx* ctx, const Plan& plan) {
  static const bool tdump = getenv("QS_PLAN_TIMING") != nullptr;  // diagnostics
  const auto te0 = std::chrono::steady_clock::now();
  // sub-state pool
  std::vector<size_t> sub_off(plan.subs.size() + 1, 0);
  size_t sub_total = 0;
  for (size_t i = 0; i < plan.subs.size(); i++) {
    sub_off[i + 1] = sub_total;
    sub_total += (size_t)1 << plan.subs[i].nq;
  }
  // encode all pass descriptors per shard
  std::vector<std::vector<size_t>> blob_off(ctx->shards.size());
  std::vector<std::vector<unsigned char>> blobs(ctx->shards.size());
  for (size_t si = 0; si < ctx->shards.size(); si++) {
    Shard& sh = ctx->shards[si];
    CU(cudaSetDevice(sh.device));
    if (sub_total > sh.subpool_cap) {
      if (sh.subpool) cudaFree(sh.subpool);
      CU(cudaMalloc(&sh.subpool, sub_total * sizeof(double2)));
      sh.subpool_cap = sub_total;
    }
    std::vector<unsigned char>& all = blobs[si];
    for (const Step& st : plan.steps) {
      size_t off = (size_t)-1;
      if (st.type == Step::PASS) {
        std::vector<unsigned char> b;
        std::string err;
        const int rank = (st.pass.buf == 0) ? sh.rank : 0;
        int rc = encode_pass(st.pass, rank, b, err);
        if (rc) return set_err(ctx, rc, err);
        KPass h;
        memcpy(&h, b.data(), sizeof h);
        if (st.pass.src_mode == 1) {
          h.expand.n = (int)st.pass.exp_bufs.size();
          for (int g = 0; g < h.expand.n; g++) {
            h.expand.ptr[g] = (u64)(sh.subpool + sub_off[st.pass.exp_bufs[g]]);
            h.expand.lo[g] = st.pass.exp_lo[g];
            h.expand.len[g] = st.pass.exp_len[g];
          }
          memcpy(b.data(), &h, sizeof h);
        }
        while (all.size() % 256) all.push_back(0);
        off = all.size();
        all.insert(all.end(), b.begin(), b.end());
      }
      blob_off[si].push_back(off);
    }
    if (all.size() > sh.arena_cap) {
      if (sh.arena) cudaFree(sh.arena);
      size_t cap = std::max(all.size() * 2, (size_t)1 << 20);
      CU(cudaMalloc(&sh.arena, cap));
      sh.arena_cap = cap;
    }
  }
  // the previous circuit (accumulating mode: still in flight) must be done
  // before its staging buffer, descriptors and events are reused; the
  // planning and encoding above overlapped it
  {
    const int rc = finish_inflight(ctx);
    if (rc) return rc;
  }
  ctx->n_fused_swaps = 0;  // per call (qs_stats_t reports the last call)
  ctx->fused_pending = false;
  size_t stage_total = 0;
  for (auto& b : blobs) stage_total += (b.size() + 255) & ~(size_t)255;
  int rc = ensure_host_stage(ctx, stage_total);
  if (rc) return rc;
  {
    size_t o = 0;
    for (size_t si = 0; si < ctx->shards.size(); si++) {
      Shard& sh = ctx->shards[si];
      if (blobs[si].empty()) continue;
      memcpy(ctx->host_stage + o, blobs[si].data(), blobs[si].size());
      CU(cudaSetDevice(sh.device));
      CU(cudaMemcpyAsync(sh.arena, ctx->host_stage + o, blobs[si].size(),
                         cudaMemcpyHostToDevice, sh.stream));
      o += (blobs[si].size() + 255) & ~(size_t)255;
    }
  }
  if (tdump) fprintf(stderr, "qs_exec encode+upload %.3f ms\n", ms_since(te0));
  // Specialised kernels for every pass are compiled (in parallel) and loaded
  // before anything launches, so a failure cannot leave a half-applied plan:
  // a pass whose kernel is not ready runs on the interpreter kernel, and a
  // swap fused into such a pass runs unfused.
  const auto tp0 = std::chrono::steady_clock::now();
  std::vector<std::vector<JitPrepared>> prep(ctx->shards.size(), std::vector<JitPrepared>(plan.steps.size()));
  std::vector<char> step_jit(plan.steps.size(), 1);  // ready on every shard
  for (size_t si = 0; si < ctx->shards.size(); si++) {
    Shard& sh = ctx->shards[si];
    std::vector<const unsigned char*> list;
    std::vector<size_t> at;
    for (size_t k = 0; k < plan.steps.size(); k++) {
      const Step& st = plan.steps[k];
      if (st.type != Step::PASS || st.pass.kernel == KK_SMALL || st.pass.nl < ctx->cfg.jit_min_qubits) {
        step_jit[k] = 0;
        continue;
      }
      list.push_back(blobs[si].data() + blob_off[si][k]);
      at.push_back(k);
    }
    if (list.empty()) continue;
    CU(cudaSetDevice(sh.device));
    std::vector<JitPrepared> res;
    jit_prepare_all(list, sh.device, res, false);
    for (size_t i = 0; i < at.size(); i++) {
      if (!res[i].ok) {
        ctx->jit_errors++;
        ctx->jit_last_error = res[i].err;
        step_jit[at[i]] = 0;
      }
      prep[si][at[i]] = std::move(res[i]);
    }
  }
  // fused swaps (f1) need the specialised kernel of the exporting pass on
  // every rank: in rank mode all ranks vote (min) so they agree
  bool any_fusable = false;
  for (size_t k = 0; k + 1 < plan.steps.size(); k++)
    if (plan.steps[k].type == Step::PASS && plan.steps[k].pass.x_j && plan.steps[k + 1].type == Step::SWAP &&
        plan.steps[k + 1].fusable)
      any_fusable = true;
  bool fuse_vote = true;
  if (any_fusable && ctx->mode == M_RANK && ctx->n_ranks > 1) {
    double v = 1.0;
    for (size_t k = 0; k < plan.steps.size(); k++)
      if (plan.steps[k].type == Step::PASS && (plan.steps[k].pass.x_j || plan.steps[k].pass.pull_j) && !step_jit[k])
        v = 0.0;
    Shard& sh = ctx->shards[0];
    CU(cudaSetDevice(sh.device));
    double* dv = reinterpret_cast<double*>(sh.bar) + 1;
    CU(cudaMemcpyAsync(dv, &v, sizeof v, cudaMemcpyHostToDevice, sh.stream));
    NC(ncclAllReduce(dv, dv, 1, ncclDouble, ncclMin, sh.comm, sh.stream));
    CU(cudaMemcpyAsync(&v, dv, sizeof v, cudaMemcpyDeviceToHost, sh.stream));
    CU(cudaStreamSynchronize(sh.stream));
    fuse_vote = v == 1.0;
  }
  auto will_fuse = [&](size_t k) {
    if (k + 1 >= plan.steps.size()) return false;
    const Step& st = plan.steps[k];
    const Step& nx = plan.steps[k + 1];
    // a split exporting pass leaves half its chunks for the next pass to
    // pull: that pass must run its specialised kernel too
    const bool split_ok = st.type != Step::PASS || st.pass.x_split < 0 ||
                          (k + 2 < plan.steps.size() && step_jit[k + 2]);
    return st.type == Step::PASS && st.pass.x_j && nx.type == Step::SWAP && nx.fusable && fuse_vote &&
           step_jit[k] && split_ok && ensure_peers(ctx) == 1;
  };
  // Co-scheduled runs (two-level blocking, f2; planner mark_l2_groups): up
  // to kMaxRun consecutive passes of an L2 group become one cooperative
  // launch (jit_prepare_run).  run_end[a] = one past the last pass of the run
  // starting at step a (0: none); every shard must have it, else the passes
  // run one by one.
  std::vector<size_t> run_end(plan.steps.size(), 0);
  std::vector<int> run_sb(plan.steps.size(), 0);
  std::vector<std::vector<JitPrepared>> run_prep(ctx->shards.size(), std::vector<JitPrepared>(plan.steps.size()));
  // (loopback shards share one device: their cooperative launches would
  // compete for the same SMs, so runs are used with one shard per device)
  if (ctx->cfg.l2_block_qubits > 0 && !getenv("QS_NO_L2RUN") &&
      (ctx->mode != M_LOOPBACK || ctx->shards.size() == 1)) {
    for (size_t a = 0; a < plan.steps.size();) {
      const Step& st = plan.steps[a];
      if (st.type != Step::PASS || st.pass.l2_grp < 0) {
        a++;
        continue;
      }
      size_t b = a;
      while (b < plan.steps.size() && b - a < (size_t)kMaxRun && plan.steps[b].type == Step::PASS &&
             plan.steps[b].pass.l2_grp == st.pass.l2_grp)
        b++;
      if (b - a >= 2) {
        int wm = kChunkBits;
        for (size_t q = a; q < b; q++) {
          for (int c : plan.steps[q].pass.cpos) wm = std::max(wm, c + 1);
          for (int c : plan.steps[q].pass.opos) wm = std::max(wm, c + 1);
        }
        bool ok = true;
        for (size_t si = 0; ok && si < ctx->shards.size(); si++) {
          std::vector<const unsigned char*> hbs;
          for (size_t q = a; q < b; q++) {
            if (!prep[si][q].ok) ok = false;
            hbs.push_back(blobs[si].data() + blob_off[si][q]);
          }
          if (!ok) break;
          CU(cudaSetDevice(ctx->shards[si].device));
          if (!jit_prepare_run(hbs, wm - kChunkBits, ctx->shards[si].device, run_prep[si][a])) {
            ok = false;
            ctx->jit_last_error = "run: " + run_prep[si][a].err;
          }
        }
        if (ok) {
          run_end[a] = b;
          run_sb[a] = wm - kChunkBits;
        }
      }
      a = b;
    }
  }
  std::vector<char> pulling(plan.steps.size(), 0);  // pull pass whose source was split
  ctx->prep_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count();
  if (tdump) fprintf(stderr, "qs_exec prep %.3f ms\n", ctx->prep_ms);
  for (Shard& sh : ctx->shards) {
    CU(cudaSetDevice(sh.device));
    sh.timed.clear();
    sh.ev_used = 0;
    CU(cudaEventRecord(sh.t0, sh.stream));
  }
  // Per-chunk tables (qs_kshape_table) depend only on the descriptors: all
  // of them are computed on a side stream right at the start, so they
  // overlap the passes before theirs instead of sitting in front of them
  // (<= 1 GiB of tables per shard; else each is computed before its pass).
  std::vector<std::vector<size_t>> tab_off(ctx->shards.size(), std::vector<size_t>(plan.steps.size(), (size_t)-1));
  std::vector<std::vector<cudaEvent_t>> tab_ev(ctx->shards.size(), std::vector<cudaEvent_t>(plan.steps.size(), nullptr));
  for (size_t si = 0; si < ctx->shards.size(); si++) {
    Shard& sh = ctx->shards[si];
    size_t total = 0;
    std::vector<TabCols> cols(plan.steps.size());
    for (size_t k = 0; k < plan.steps.size(); k++) {
      if (!prep[si][k].ok) continue;
      const unsigned char* hb = blobs[si].data() + blob_off[si][k];
      if (!jit_table_cols(hb, &cols[k])) continue;
      KPass h;
      memcpy(&h, hb, sizeof h);
      tab_off[si][k] = total;
      total += ((size_t)h.n_chunks * cols[k].width + 31) & ~(size_t)31;
    }
    if (total == 0) continue;
    if (total * sizeof(u64) > ((size_t)1 << 30)) {  // too much: tables per pass
      for (size_t k = 0; k < plan.steps.size(); k++) tab_off[si][k] = (size_t)-1;
      continue;
    }
    CU(cudaSetDevice(sh.device));
    if (!sh.side) CU(cudaStreamCreateWithFlags(&sh.side, cudaStreamNonBlocking));
    if (total > sh.vtab_cap) {
      if (sh.vtab) CU(cudaFree(sh.vtab));
      sh.vtab = nullptr;
      sh.vtab_cap = 0;
      CU(cudaMalloc(&sh.vtab, total * sizeof(u64)));
      sh.vtab_cap = total;
    }
    CU(cudaStreamWaitEvent(sh.side, sh.t0, 0));
    for (size_t k = 0; k < plan.steps.size(); k++) {
      if (tab_off[si][k] == (size_t)-1) continue;
      const unsigned char* hb = blobs[si].data() + blob_off[si][k];
      KPass h;
      memcpy(&h, hb, sizeof h);
      CU(launch_shape_table(sh.arena + blob_off[si][k], sh.vtab + tab_off[si][k], h.rank_base, h.n_chunks, cols[k],
                            sh.side));
      ctx->launches++;
      tab_ev[si][k] = get_event(sh);
      CU(cudaEventRecord(tab_ev[si][k], sh.side));
    }
  }
  const size_t shard_amps = (size_t)1 << ctx->nl;
  for (size_t k = 0; k < plan.steps.size(); k++) {
    const Step& st = plan.steps[k];
    if (st.type == Step::SWAP) {
      Shard& s0 = ctx->shards[0];
      cudaEvent_t a = nullptr, b = nullptr;
      if (ctx->timing) {
        CU(cudaSetDevice(s0.device));
        a = get_event(s0);
        b = get_event(s0);
        CU(cudaEventRecord(a, s0.stream));
      }
      if (st.fusable && ctx->fused_pending) {
        // the preceding pass already stored every piece in its destination's
        // receive buffer: wait for all of them, then the buffers trade roles
        rc = shard_barrier(ctx);
        if (rc) return rc;
        for (Shard& sh : ctx->shards) std::swap(sh.state, sh.scratch);
        ctx->n_fused_swaps++;
      } else if (top_lpos(ctx, st)) {
        rc = exec_swap(ctx, st);
        if (rc) return rc;
      } else {
        // a direct swap planned for fusion but run unfused (no peer access):
        // transpose lpos[i] <-> top[i], swap the top positions, transpose back
        Step tst = st;
        std::vector<int> ta, tb;
        for (int i = 0; i < st.j; i++) {
          tst.lpos[i] = ctx->nl - st.j + i;
          if (st.lpos[i] != tst.lpos[i]) ta.push_back(st.lpos[i]), tb.push_back(tst.lpos[i]);
        }
        for (int pass = 0; pass < 3; pass++) {
          if (pass == 1) {
            rc = exec_swap(ctx, tst);
            if (rc) return rc;
            ctx->swap_parity++;
            continue;
          }
          for (Shard& sh : ctx->shards) {
            CU(cudaSetDevice(sh.device));
            CU(launch_permute(sh.state, sh.scratch, shard_amps, ta.data(), tb.data(), (int)ta.size(), sh.stream));
            std::swap(sh.state, sh.scratch);
            ctx->launches++;
          }
          ctx->swap_parity++;
        }
        ctx->swap_parity--;  // the step's own increment follows
      }
      ctx->fused_pending = false;
      ctx->swap_parity++;
      if (ctx->timing) {
        CU(cudaSetDevice(s0.device));
        CU(cudaEventRecord(b, s0.stream));
        s0.timed.push_back({KK_SWAP, a, b, (uint64_t)((16ull << ctx->nl) - (16ull << (ctx->nl - st.j)))});
      }
      continue;
    }
    // A pass that stores into its peers' receive buffers may only start
    // once every peer is done with all earlier steps (an unfused swap's
    // local copy or a permute may still read the buffer that is now the
    // peer's receive buffer).
    // Two-level blocking: a co-scheduled run of passes in
    // one cooperative launch (jit_prepare_run); its per-chunk tables were
    // computed ahead on the side stream (else the passes run one by one).
    if (st.type == Step::PASS && run_end[k]) {
      const size_t k1 = run_end[k];
      bool ok = true;
      for (size_t si = 0; ok && si < ctx->shards.size(); si++)
        for (size_t q = k; ok && q < k1; q++) {
          TabCols vl;
          if (tab_off[si][q] == (size_t)-1 && jit_table_cols(blobs[si].data() + blob_off[si][q], &vl)) ok = false;
        }
      if (ok) {
        const int K = (int)(k1 - k);
        for (size_t si = 0; si < ctx->shards.size(); si++) {
          Shard& sh = ctx->shards[si];
          CU(cudaSetDevice(sh.device));
          cudaEvent_t a = nullptr, b = nullptr;
          if (ctx->timing) {
            a = get_event(sh);
            b = get_event(sh);
            CU(cudaEventRecord(a, sh.stream));
          }
          std::vector<const unsigned char*> dbs, hbs;
          std::vector<const u64*> vts;
          u64 n_chunks = 0;
          for (size_t q = k; q < k1; q++) {
            dbs.push_back(sh.arena + blob_off[si][q]);
            hbs.push_back(blobs[si].data() + blob_off[si][q]);
            KPass h;
            memcpy(&h, hbs.back(), sizeof h);
            n_chunks = h.n_chunks;
            const u64* vt = sh.vtab;
            if (tab_off[si][q] != (size_t)-1) {
              vt = sh.vtab + tab_off[si][q];
              CU(cudaStreamWaitEvent(sh.stream, tab_ev[si][q], 0));
            }
            vts.push_back(vt);
          }
          const JitPrepared& rp = run_prep[si][k];
          const unsigned nblk = (unsigned)(n_chunks >> run_sb[k]);
          const size_t fbytes = (size_t)K * nblk * sizeof(unsigned);
          if (fbytes > sh.l2flags_cap) {
            if (sh.l2flags) CU(cudaFree(sh.l2flags));
            sh.l2flags = nullptr;
            sh.l2flags_cap = 0;
            CU(cudaMalloc(&sh.l2flags, fbytes));
            sh.l2flags_cap = fbytes;
          }
          CU(cudaMemsetAsync(sh.l2flags, 0, fbytes, sh.stream));
          // the CTAs are dealt to the members by weight (QS_L2_SPLIT:
          // comma-separated weights; default equal), each share a multiple
          // of the members' grid multiple where possible
          const int grid = num_sms_of(sh.device) * rp.per_sm;
          std::vector<double> w(K, 1.0);
          if (const char* e = getenv("QS_L2_SPLIT")) {
            const char* c = e;
            for (int i = 0; i < K && *c; i++) {
              w[i] = atof(c);
              while (*c && *c != ',') c++;
              if (*c == ',') c++;
            }
          }
          double wsum = 0;
          for (double x : w) wsum += x;
          unsigned split[kMaxRun];
          unsigned at = 0;
          for (int i = 0; i < K; i++) {
            unsigned n_i = (unsigned)(grid * w[i] / wsum);
            if (rp.grid_mult > 1 && n_i > (unsigned)rp.grid_mult) n_i -= n_i % (unsigned)rp.grid_mult;
            if (n_i < 1) n_i = 1;
            if (i == K - 1 || at + n_i > (unsigned)grid - (unsigned)(K - 1 - i)) n_i = (unsigned)grid - at - (unsigned)(K - 1 - i);
            at += n_i;
            split[i] = at;
          }
          // the first pass may run this far (QS_L2_LAG MiB, default 24) ahead
          // of the last one
          static const double lag_mib = getenv("QS_L2_LAG") ? atof(getenv("QS_L2_LAG")) : 24.0;
          const double blk_mib = (double)(16ull << (kChunkBits + run_sb[k])) / (1 << 20);
          // The lag must exceed what the members have in flight together: a
          // member's ring loads up to 3 chunks of its CTA sequence ahead
          // (3 x its CTA count in chunk order) before it finishes a chunk,
          // and each member's loads wait for the one before it; with less
          // lag the first member's throttle and the prefetches wait for each
          // other.  Per member: 4 rounds of its CTAs, rounded up to blocks,
          // plus one block.
          unsigned min_lag = 1;
          for (int i = 0; i < K; i++) {
            const unsigned nb_i = split[i] - (i ? split[i - 1] : 0u);
            min_lag += ((4u * nb_i + (1u << run_sb[k]) - 1u) >> run_sb[k]) + 1u;
          }
          const unsigned lag = std::max(min_lag, (unsigned)std::max(1.0, lag_mib / blk_mib));
          CU(jit_launch_run(rp, grid, dbs, hbs, sh.state, (u64)sh.rank << ctx->nl, vts, n_chunks, sh.l2flags, nblk,
                            split, lag, sh.stream));
          ctx->launches += 2;
          ctx->jit_launches++;
          ctx->jit_variant[rp.variant]++;
          if (ctx->timing) {
            CU(cudaEventRecord(b, sh.stream));
            const PassPlan& p0 = plan.steps[k].pass;
            sh.timed.push_back({KK_L2, a, b, (uint64_t)((p0.src_mode ? 16ull : 32ull) << ctx->nl)});
          }
        }
        ctx->n_l2_groups++;
        k = k1 - 1;
        continue;
      }
    }
    const bool fuse = will_fuse(k);
    if (fuse) {
      rc = shard_barrier(ctx);
      if (rc) return rc;
      if (st.pass.x_split >= 0) pulling[k + 2] = 1;
    }
    for (size_t si = 0; si < ctx->shards.size(); si++) {
      Shard& sh = ctx->shards[si];
      CU(cudaSetDevice(sh.device));
      cudaEvent_t a = nullptr, b = nullptr;
      const bool tm = ctx->timing;
      if (tm) {
        a = get_event(sh);
        b = get_event(sh);
        CU(cudaEventRecord(a, sh.stream));
      }
      int kind = KK_INIT;
      uint64_t bytes = 0;
      switch (st.type) {
        case Step::INIT_BASIS: {
          CU(cudaMemsetAsync(sh.state, 0, shard_amps * sizeof(double2), sh.stream));
          ctx->launches++;
          if ((st.basis >> ctx->nl) == (u64)sh.rank) {
            CU(launch_set_one(sh.state, st.basis & (shard_amps - 1), sh.stream));
            ctx->launches++;
          }
          kind = KK_INIT;
          bytes = 16ull << ctx->nl;
          break;
        }
        case Step::SUB_INIT: {
          double2* d = sh.subpool + sub_off[st.buf];
          const size_t na = (size_t)1 << plan.subs[st.buf - 1].nq;
          CU(cudaMemsetAsync(d, 0, na * sizeof(double2), sh.stream));
          CU(launch_set_one(d, st.basis, sh.stream));
          ctx->launches += 2;
          kind = KK_INIT;
          bytes = 16ull * na;
          break;
        }
        case Step::SUB_MERGE: {
          double2* d = sh.subpool + sub_off[st.buf];
          const int la = plan.subs[st.src_a - 1].nq, lb = plan.subs[st.src_b - 1].nq;
          CU(launch_merge(d, sh.subpool + sub_off[st.src_a], la, sh.subpool + sub_off[st.src_b], lb,
                          sh.stream));
          ctx->launches++;
          kind = KK_MERGE;
          bytes = 16ull << (la + lb);
          break;
        }
        case Step::PERMUTE: {
          CU(launch_permute(sh.state, sh.scratch, shard_amps, st.gpos.data(), st.lpos.data(),
                            (int)st.gpos.size(), sh.stream));
          std::swap(sh.state, sh.scratch);
          if (si == 0) ctx->swap_parity++;
          ctx->launches++;
          kind = KK_SWAP;
          bytes = 32ull << ctx->nl;
          break;
        }
        case Step::EXPAND: {
          KExpand e;
          memset(&e, 0, sizeof e);
          e.n = (int)st.exp_bufs.size();
          for (int g = 0; g < e.n; g++) {
            e.ptr[g] = (u64)(sh.subpool + sub_off[st.exp_bufs[g]]);
            e.lo[g] = st.exp_lo[g];
            e.len[g] = st.exp_len[g];
          }
          CU(launch_expand(sh.state, shard_amps, (u64)sh.rank << ctx->nl, e, sh.stream));
          ctx->launches++;
          kind = KK_EXPAND;
          bytes = 16ull << ctx->nl;
          break;
        }
        case Step::PASS: {
          const PassPlan& p = st.pass;
          const unsigned char* dblob = sh.arena + blob_off[si][k];
          KPass h;
          memcpy(&h, blobs[si].data() + blob_off[si][k], sizeof h);
          double2* buf = (p.buf == 0) ? sh.state : (sh.subpool + sub_off[p.buf]);
          // fused swap: this pass exports the next swap's pieces (decided the
          // same way on every shard and rank: plan, kernel readiness vote,
          // collective peer setup); otherwise every destination is our own
          // buffer at our own index
          u64 xp[2 << kMaxXBits];
          for (int s = 0; s < (2 << kMaxXBits); s++) xp[s] = (u64)buf;
          if (fuse) {
            fused_targets(ctx, plan.steps[k + 1], sh.rank, xp);
            ctx->fused_pending = true;
          }
          if (pulling[k]) {
            // pull pass: elements of chunks with the split bit set come from
            // the buffer the exporting pass left them in, at the source rank
            // of their piece (the swap's formula with the roles of the two
            // allocations exchanged: recv_buffer is now each rank's old state)
            fused_targets(ctx, plan.steps[k - 1], sh.rank, xp + (1 << kMaxXBits));
          }
          const JitPrepared& jp = prep[si][k];
          if (jp.ok) {
            void* fn = jp.fn;
            const int per_sm = jp.per_sm;
            const size_t smem = jp.smem;
            u64 grid = (u64)num_sms_of(sh.device) * per_sm;
            // with QS_JIT_WO_MINB (A/B knob) keep grids a multiple of 8 so the
            // hoisted expand gathers stay enabled at 3 CTAs per SM
            if (getenv("QS_JIT_WO_MINB") && per_sm != 2 && grid > 8) grid &= ~7ull;
            if (jp.grid_mult > 1 && grid > (u64)jp.grid_mult) grid -= grid % (u64)jp.grid_mult;
            if (grid > h.n_chunks) grid = h.n_chunks;
            const unsigned char* hb = blobs[si].data() + blob_off[si][k];
            const size_t pb = jit_param_bytes(hb);
            TabCols vl;
            u64* vtab = sh.vtab;
            if (tab_off[si][k] != (size_t)-1) {
              vtab = sh.vtab + tab_off[si][k];  // computed ahead on the side stream
              CU(cudaStreamWaitEvent(sh.stream, tab_ev[si][k], 0));
            } else if (jit_table_cols(hb, &vl)) {
              const size_t need = (size_t)h.n_chunks * vl.width;
              if (need > sh.vtab_cap) {
                if (sh.vtab) CU(cudaFree(sh.vtab));
                sh.vtab = nullptr;
                sh.vtab_cap = 0;
                CU(cudaMalloc(&sh.vtab, need * sizeof(u64)));
                sh.vtab_cap = need;
              }
              CU(launch_shape_table(dblob, sh.vtab, h.rank_base, h.n_chunks, vl, sh.stream));
              ctx->launches++;
              vtab = sh.vtab;
            }
            CU(jit_launch(fn, (int)grid, smem, dblob, hb, buf, h.rank_base, vtab, xp, hb + h.off_pool,
                          pb, sh.stream, 0, h.n_chunks));
            ctx->jit_launches++;
            ctx->jit_variant[jp.variant]++;
          } else {
            // interpreter kernel (small passes, jit_min_qubits, or a kernel
            // that failed to build): stores locally, never fused
            CU(launch_pass(p.kernel, dblob, h, buf, sh.stream));
          }
          ctx->launches++;
          kind = (p.buf != 0) ? KK_SUB : fuse ? KK_XPASS : pulling[k] ? KK_PULL : p.kernel;
          bytes = ((p.src_mode ? 16ull : 32ull) << p.nl);
          break;
        }
        default:
          break;
      }
      if (tm) {
        CU(cudaEventRecord(b, sh.stream));
        sh.timed.push_back({kind, a, b, bytes});
      }
    }
    // nobody may overwrite a buffer another rank is still pulling from
    if (pulling[k]) {
      rc = shard_barrier(ctx);
      if (rc) return rc;
    }
  }
  if (tdump) fprintf(stderr, "qs_exec launched %.3f ms after execute()\n", ms_since(te0));
  for (Shard& sh : ctx->shards) {
    CU(cudaSetDevice(sh.device));
    CU(cudaEventRecord(sh.t1, sh.stream));
  }
  ctx->inflight = true;
  // In the accumulating timing mode (qs_set_timing 2, a loop of circuits)
  // the call returns once everything is enqueued: the next call's planning
  // and encoding overlap this circuit's device work, and the completion is
  // taken at the next call or at any query (finish_inflight).
  if (ctx->accumulate) return QS_OK;
  return finish_inflight(ctx);
}

// Wait for the enqueued circuit, then account its device time and per-kernel
// timings (execute_steps).  A device error found here poisons the handle.
int finish_inflight(qs_ctx* ctx) {
  if (!ctx->inflight) return QS_OK;
  ctx->inflight = false;
  static const bool tdump = getenv("QS_PLAN_TIMING") != nullptr;  // diagnostics
  for (Shard& sh : ctx->shards) {
    CU(cudaSetDevice(sh.device));
    CU(cudaStreamSynchronize(sh.stream));
    CU(cudaGetLastError());
  }
  // timing
  double tdev = 0;
  for (Shard& sh : ctx->shards) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, sh.t0, sh.t1));
    if (ms > tdev) tdev = ms;
  }
  if (ctx->accumulate) {
    ctx->stats.t_device_ms += tdev;
  } else {
    ctx->stats.t_device_ms = tdev;
    memset(ctx->k_count, 0, sizeof ctx->k_count);
    memset(ctx->k_ms, 0, sizeof ctx->k_ms);
    memset(ctx->k_bytes, 0, sizeof ctx->k_bytes);
  }
  double tswap = 0;
  if (ctx->timing) {
    Shard& s0 = ctx->shards[0];
    static const bool dump = getenv("QS_TIMING_DUMP") != nullptr;  // per-launch times (diagnostics)
    for (const Timed& t : s0.timed) {
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, t.a, t.b));
      if (dump) fprintf(stderr, "qs_timing rank %d kind %d ms %.4f bytes %llu\n", s0.rank, t.kind, ms,
                        (unsigned long long)t.bytes);
      ctx->k_count[t.kind]++;
      ctx->k_ms[t.kind] += ms;
      ctx->k_bytes[t.kind] += t.bytes;
      if (t.kind == KK_SWAP) tswap += ms;
    }
  }
  ctx->stats.t_swap_ms = tswap;
  ctx->stats.n_fused_swaps = ctx->n_fused_swaps;
  if (tdump) fprintf(stderr, "qs_exec done (device %.3f ms)\n", tdev);
  return QS_OK;
}

int materialize(qs_ctx* ctx) {
  if (!ctx->pending) return QS_OK;
  return qs_apply_circuit(ctx, nullptr, 0);
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

void qs_default_config(qs_config_t* cfg) {
  cfg->chunk_qubits = kChunkBits;
  cfg->fuse_cap = 4;
  cfg->diag_cap = 0;
  cfg->boost_div = 2;
  cfg->flags = QS_OPT_ALL;
  cfg->jit_min_qubits = jit_default_min();
  // two-level blocking (f2) is off by default: on QFT-30 the co-scheduled
  // run measured 15.8 ms against 9.2 ms pass by pass
  static const int l2b = getenv("QS_L2_BLOCK") ? atoi(getenv("QS_L2_BLOCK")) : 0;
  cfg->l2_block_qubits = l2b;
}

static int create_common(qs_ctx* ctx) {
  for (Shard& s : ctx->shards) {
    int rc = alloc_shard_memory(ctx, s);
    if (rc) return rc;
  }
  return QS_OK;
}

int qs_create(int n_qubits, int n_gpus, qs_ctx** out) {
  if (!out) return QS_EINVAL;
  *out = nullptr;
  std::string why;
  if (check_dims(n_qubits, n_gpus, why)) return QS_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return QS_ECUDA;
  if (n_gpus > ndev) return QS_EINVAL;
  qs_ctx* ctx = new qs_ctx();
  *out = ctx;
  init_ctx(ctx, n_qubits, n_gpus);
  ctx->mode = M_SINGLE;
  ctx->shards.resize(n_gpus);
  for (int r = 0; r < n_gpus; r++) {
    Shard& s = ctx->shards[r];
    s.device = r;
    s.rank = r;
    CU(cudaSetDevice(r));
    CU(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    s.own_stream = true;
  }
  if (n_gpus > 1) {
    std::vector<ncclComm_t> comms(n_gpus);
    std::vector<int> devs(n_gpus);
    for (int r = 0; r < n_gpus; r++) devs[r] = r;
    NC(ncclCommInitAll(comms.data(), n_gpus, devs.data()));
    for (int r = 0; r < n_gpus; r++) ctx->shards[r].comm = comms[r];
  }
  int rc = create_common(ctx);
  if (rc) return rc;
  return QS_OK;
}

int qs_create_loopback(int n_qubits, int n_ranks, int device, qs_ctx** out) {
  if (!out) return QS_EINVAL;
  *out = nullptr;
  std::string why;
  if (check_dims(n_qubits, n_ranks, why)) return QS_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return QS_ECUDA;
  if (device < 0 || device >= ndev) return QS_EINVAL;
  qs_ctx* ctx = new qs_ctx();
  *out = ctx;
  init_ctx(ctx, n_qubits, n_ranks);
  ctx->mode = M_LOOPBACK;
  ctx->shards.resize(n_ranks);
  CU(cudaSetDevice(device));
  cudaStream_t st;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (int r = 0; r < n_ranks; r++) {
    Shard& s = ctx->shards[r];
    s.device = device;
    s.rank = r;
    s.stream = st;
    s.own_stream = (r == 0);
  }
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const size_t need = ((size_t)16 << ctx->nl) * 2 * n_ranks;
  if (need > fr) return set_err(ctx, QS_ENOMEM, "loopback needs " + std::to_string(need) + " bytes");
  return create_common(ctx);
}

int qs_nccl_unique_id(void* id_out_128) {
  if (!id_out_128) return QS_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return QS_ENCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  memcpy(id_out_128, &id, 128);
  return QS_OK;
}

int qs_create_rank(int n_qubits, int world_size, int rank, int device, const void* nccl_id_128,
                   qs_ctx** out) {
  if (!out) return QS_EINVAL;
  *out = nullptr;
  std::string why;
  if (check_dims(n_qubits, world_size, why)) return QS_EINVAL;
  if (rank < 0 || rank >= world_size) return QS_EINVAL;
  if (world_size > 1 && !nccl_id_128) return QS_EINVAL;
  qs_ctx* ctx = new qs_ctx();
  *out = ctx;
  init_ctx(ctx, n_qubits, world_size);
  ctx->mode = M_RANK;
  ctx->shards.resize(1);
  Shard& s = ctx->shards[0];
  s.device = device;
  s.rank = rank;
  CU(cudaSetDevice(device));
  CU(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  s.own_stream = true;
  if (world_size > 1) {
    ncclUniqueId id;
    memcpy(&id, nccl_id_128, 128);
    NC(ncclCommInitRank(&s.comm, world_size, id, rank));
  }
  return create_common(ctx);
}

void qs_destroy(qs_ctx* ctx) {
  if (!ctx) return;
  for (Shard& s : ctx->shards) {  // loopback shards share one stream: sync all first
    cudaSetDevice(s.device);
    if (s.stream) cudaStreamSynchronize(s.stream);
  }
  if (ctx->mode == M_RANK && !ctx->ipc.empty()) {
    cudaSetDevice(ctx->shards[0].device);
    for (int r = 0; r < ctx->n_ranks; r++)
      if (r != ctx->shards[0].rank)
        for (int k = 0; k < 2; k++)
          if (ctx->ipc[2 * r + k]) cudaIpcCloseMemHandle(ctx->ipc[2 * r + k]);
  }
  for (Shard& s : ctx->shards) {
    cudaSetDevice(s.device);
    if (s.comm) ncclCommDestroy(s.comm);
    cudaFree(s.state);
    cudaFree(s.scratch);
    cudaFree(s.arena);
    cudaFree(s.subpool);
    cudaFree(s.tmp);
    cudaFree(s.dmap);
    cudaFree(s.vtab);
    cudaFree(s.l2flags);
    cudaFree(s.bar);
    for (cudaEvent_t e : s.ev_pool) cudaEventDestroy(e);
    if (s.t0) cudaEventDestroy(s.t0);
    if (s.t1) cudaEventDestroy(s.t1);
    if (s.own_stream && s.stream) cudaStreamDestroy(s.stream);
    if (s.side) cudaStreamDestroy(s.side);
  }
  if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
  if (ctx->host_tmp) cudaFreeHost(ctx->host_tmp);
  delete ctx;
}

int qs_set_config(qs_ctx* ctx, const qs_config_t* cfg) {
  if (!ctx || !cfg) return QS_EINVAL;
  if (cfg->chunk_qubits != kChunkBits)
    return set_err(ctx, QS_EINVAL, "chunk_qubits must be 12 in this build");
  if (cfg->fuse_cap < 1 || cfg->fuse_cap > 4) return set_err(ctx, QS_EINVAL, "fuse_cap in [1,4]");
  if (cfg->diag_cap < 0 || cfg->diag_cap > 64) return set_err(ctx, QS_EINVAL, "diag_cap in [0,64]");
  if (cfg->boost_div < 1 || cfg->boost_div > 64) return set_err(ctx, QS_EINVAL, "boost_div in [1,64]");
  if (cfg->flags & ~QS_OPT_ALL) return set_err(ctx, QS_EINVAL, "unknown flags");
  if (cfg->jit_min_qubits < 0) return set_err(ctx, QS_EINVAL, "jit_min_qubits >= 0");
  if (cfg->l2_block_qubits != 0 && (cfg->l2_block_qubits < 14 || cfg->l2_block_qubits > 40))
    return set_err(ctx, QS_EINVAL, "l2_block_qubits 0 or in [14,40]");
  ctx->cfg = *cfg;
  return QS_OK;
}

int qs_get_config(const qs_ctx* ctx, qs_config_t* cfg) {
  if (!ctx || !cfg) return QS_EINVAL;
  *cfg = ctx->cfg;
  return QS_OK;
}

int qs_set_basis_state(qs_ctx* ctx, uint64_t x) {
  if (!ctx) return QS_EINVAL;
  if (ctx->poisoned) return QS_EPOISONED;
  if (ctx->n < 64 && (x >> ctx->n)) return set_err(ctx, QS_EINVAL, "basis index >= 2^n");
  ctx->pending = true;
  ctx->basis = x;
  for (int q = 0; q < ctx->n; q++) ctx->map[q] = q;
  return QS_OK;
}

int qs_apply_circuit(qs_ctx* ctx, const qs_gate_t* gates, size_t n_gates) {
  if (!ctx) return QS_EINVAL;
  if (ctx->poisoned) return set_err(ctx, QS_EPOISONED, "handle poisoned by an earlier device error");
  if (n_gates && !gates) return set_err(ctx, QS_EINVAL, "gates == NULL");
  auto t0 = std::chrono::steady_clock::now();
  std::vector<IrGate> ir;
  std::string err;
  int rc = ingest(ctx->n, gates, n_gates, ir, err);
  if (rc) return set_err(ctx, rc, err);
  PlanInput in;
  in.n = ctx->n;
  in.n_global = ctx->n_global;
  in.cfg = ctx->cfg;
  in.product_state = ctx->pending;
  in.basis = ctx->basis;
  in.map = ctx->map;
  auto tin = std::chrono::steady_clock::now();
  Plan plan;
  rc = make_plan(in, ir, plan, err);
  if (rc) return set_err(ctx, rc, err);
  auto t1 = std::chrono::steady_clock::now();
  static const bool tdump = getenv("QS_PLAN_TIMING") != nullptr;  // diagnostics
  if (tdump)
    fprintf(stderr, "qs_apply ingest %.3f ms, plan %.3f ms\n",
            std::chrono::duration<double, std::milli>(tin - t0).count(),
            std::chrono::duration<double, std::milli>(t1 - tin).count());
  if (!ctx->accumulate) ctx->launches = 0;
  rc = execute(ctx, plan);
  if (rc) return rc;
  ctx->map = plan.map_out;
  ctx->pending = false;
  qs_stats_t& s = ctx->stats;
  const PlanStats& ps = plan.stats;
  s.n_gates_in = ps.n_gates_in;
  s.n_passes = ps.n_passes;
  s.n_chunk_passes = ps.n_chunk;
  s.n_dense_passes = ps.n_dense;
  s.n_diag_passes = ps.n_diag;
  s.n_small_passes = ps.n_small;
  s.n_expand = ps.n_expand;
  s.n_swaps = ps.n_swaps;
  s.n_substate_gates = ps.n_sub_gates;
  s.n_fused_diag = ps.n_fused_diag;
  s.bytes_hbm = ps.bytes_hbm;
  s.bytes_nvlink = ps.bytes_nvlink;
  s.paper_updates = ps.paper_updates;
  s.naive_updates = ps.naive_updates;
  const double tp = std::chrono::duration<double, std::milli>(t1 - t0).count();
  s.t_plan_ms = ctx->accumulate ? s.t_plan_ms + tp : tp;
  return QS_OK;
}

static int readout(qs_ctx* ctx, double* host_out, uint64_t offset, uint64_t count, int probs) {
  if (!ctx || (!host_out && count)) return QS_EINVAL;
  if (ctx->poisoned) return set_err(ctx, QS_EPOISONED, "handle poisoned");
  const uint64_t total = (ctx->n >= 64) ? ~0ull : (1ull << ctx->n);
  if (offset > total || count > total - offset) return set_err(ctx, QS_EINVAL, "range exceeds 2^n");
  int rc = materialize(ctx);
  if (rc) return rc;
  const int per = probs ? 1 : 2;
  const uint64_t slice = (uint64_t)1 << 22;
  const size_t need_host = (size_t)std::min<uint64_t>(slice, std::max<uint64_t>(count, 1)) * 2;
  if (ctx->host_tmp_cap < need_host) {
    if (ctx->host_tmp) cudaFreeHost(ctx->host_tmp);
    CU(cudaMallocHost(&ctx->host_tmp, need_host * sizeof(double)));
    ctx->host_tmp_cap = need_host;
  }
  int8_t hmap[64];
  memset(hmap, 0, sizeof hmap);
  for (int q = 0; q < ctx->n; q++) hmap[q] = (int8_t)ctx->map[q];
  for (Shard& sh : ctx->shards) {
    CU(cudaSetDevice(sh.device));
    if (sh.tmp_cap < slice) {
      if (sh.tmp) cudaFree(sh.tmp);
      CU(cudaMalloc(&sh.tmp, slice * sizeof(double2)));
      sh.tmp_cap = slice;
    }
    CU(cudaMemcpyAsync(sh.dmap, hmap, 64, cudaMemcpyHostToDevice, sh.stream));
  }
  // One shard per process (rank mode, or a single GPU): the slice goes
  // straight into the caller's buffer (a DMA when the buffer is pinned).
  // Several shards in this process: each gathers its part (zeros elsewhere)
  // and the host sums them.
  const bool direct = ctx->mode == M_RANK || ctx->shards.size() == 1;
  if (!direct) memset(host_out, 0, count * per * sizeof(double));
  for (uint64_t done = 0; done < count; done += slice) {
    const uint64_t c = std::min(slice, count - done);
    if (direct) {
      Shard& sh = ctx->shards[0];
      CU(cudaSetDevice(sh.device));
      CU(launch_gather(sh.state, sh.tmp, offset + done, c, ctx->n, sh.dmap, ctx->nl,
                       (u64)sh.rank, probs, sh.stream));
      if (ctx->mode == M_RANK && ctx->n_ranks > 1)
        NC(ncclAllReduce(sh.tmp, sh.tmp, c * per, ncclDouble, ncclSum, sh.comm, sh.stream));
      CU(cudaMemcpyAsync(host_out + done * per, sh.tmp, c * per * sizeof(double),
                         cudaMemcpyDeviceToHost, sh.stream));
      CU(cudaStreamSynchronize(sh.stream));
    } else {
      for (Shard& sh : ctx->shards) {
        CU(cudaSetDevice(sh.device));
        CU(launch_gather(sh.state, sh.tmp, offset + done, c, ctx->n, sh.dmap, ctx->nl,
                         (u64)sh.rank, probs, sh.stream));
        CU(cudaMemcpyAsync(ctx->host_tmp, sh.tmp, c * per * sizeof(double),
                           cudaMemcpyDeviceToHost, sh.stream));
        CU(cudaStreamSynchronize(sh.stream));
        double* o = host_out + done * per;
        for (uint64_t i = 0; i < c * per; i++) o[i] += ctx->host_tmp[i];
      }
    }
  }
  return QS_OK;
}

int qs_get_state(qs_ctx* ctx, double* host_out, uint64_t offset, uint64_t count) {
  if (ctx) {
    const int rc = finish_inflight(ctx);
    if (rc) return rc;
  }
  return readout(ctx, host_out, offset, count, 0);
}

int qs_probabilities(qs_ctx* ctx, double* host_out, uint64_t offset, uint64_t count) {
  if (ctx) {
    const int rc = finish_inflight(ctx);
    if (rc) return rc;
  }
  return readout(ctx, host_out, offset, count, 1);
}

int qs_get_stats(const qs_ctx* ctx, qs_stats_t* out) {
  if (!ctx || !out) return QS_EINVAL;
  {
    const int rc = finish_inflight(const_cast<qs_ctx*>(ctx));
    if (rc) return rc;
  }
  *out = ctx->stats;
  return QS_OK;
}

const char* qs_last_error(const qs_ctx* ctx) { return ctx ? ctx->err.c_str() : "NULL handle"; }

int64_t qs_plan_json(int n_qubits, int n_ranks, const qs_config_t* cfg, int product_state,
                     uint64_t basis, const qs_gate_t* gates, size_t n_gates, int detail,
                     char* buf, size_t cap) {
  std::string err;
  auto fail = [&](int rc) -> int64_t {
    if (buf && cap) {
      size_t k = std::min(cap - 1, err.size());
      memcpy(buf, err.data(), k);
      buf[k] = 0;
    }
    return rc;
  };
  if (check_dims(n_qubits, n_ranks, err)) return fail(QS_EINVAL);
  std::vector<IrGate> ir;
  int rc = ingest(n_qubits, gates, n_gates, ir, err);
  if (rc) return fail(rc);
  PlanInput in;
  in.n = n_qubits;
  in.n_global = log2i(n_ranks);
  if (cfg) in.cfg = *cfg;
  else qs_default_config(&in.cfg);
  in.product_state = product_state != 0;
  in.basis = basis;
  in.map.resize(n_qubits);
  for (int q = 0; q < n_qubits; q++) in.map[q] = q;
  Plan plan;
  rc = make_plan(in, ir, plan, err);
  if (rc) return fail(rc);
  // also validate that every pass encodes
  std::vector<std::vector<unsigned char>> blobs;
  for (const Step& st : plan.steps)
    if (st.type == Step::PASS) {
      std::vector<unsigned char> b;
      rc = encode_pass(st.pass, 0, b, err);
      if (rc) return fail(rc);
      if (detail >= 2 && st.pass.kernel != KK_SMALL) blobs.push_back(std::move(b));
    }
  if (!blobs.empty()) {
    // compile the specialised kernels (NVRTC works without a GPU), in parallel
    std::vector<const unsigned char*> list;
    for (auto& b : blobs) list.push_back(b.data());
    std::vector<JitPrepared> res;
    if (jit_prepare_all(list, 0, res, true)) {
      for (auto& r : res)
        if (!r.ok) err = r.err;
      return fail(QS_EINVAL);
    }
  }
  std::string js = plan_to_json(plan, detail != 0);
  if (buf && cap) {
    size_t k = std::min(cap - 1, js.size());
    memcpy(buf, js.data(), k);
    buf[k] = 0;
  }
  return (int64_t)js.size();
}

int qs_divider(int n, int div_size, int* out, int cap) {
  if (n < 1 || div_size < 1 || !out) return QS_EINVAL;
  std::vector<int> q;
  divider(n, div_size, q);
  if ((int)q.size() > cap) return QS_EINVAL;
  for (size_t i = 0; i < q.size(); i++) out[i] = q[i];
  return (int)q.size();
}

uint64_t qs_last_launches(const qs_ctx* ctx) { return ctx ? ctx->launches : 0; }

int64_t qs_jit_info(const qs_ctx* ctx, char* buf, size_t cap) {
  double ms = 0;
  uint64_t nc = 0, hits = 0;
  jit_stats(&ms, &nc, &hits);
  char b[768];
  std::string last = ctx ? ctx->jit_last_error.substr(0, 200) : "";
  for (char& c : last)
    if (c == '"' || c == '\\' || c == '\n' || (unsigned char)c < 32) c = ' ';
  const uint64_t* v = ctx ? ctx->jit_variant : nullptr;
  snprintf(b, sizeof b,
           "{\"jit_launches\":%llu,\"jit_errors\":%llu,\"compile_ms\":%.1f,\"compiles\":%llu,"
           "\"disk_hits\":%llu,\"prep_ms\":%.2f,\"variants\":{\"write_only\":%llu,\"bulk_tma\":%llu,"
           "\"tensor_tma\":%llu,\"cp_async\":%llu},\"l2_groups\":%llu,\"last_error\":\"%s\"}",
           (unsigned long long)(ctx ? ctx->jit_launches : 0),
           (unsigned long long)(ctx ? ctx->jit_errors : 0), ms, (unsigned long long)nc,
           (unsigned long long)hits, ctx ? ctx->prep_ms : 0.0,
           (unsigned long long)(v ? v[JV_WRITE_ONLY] : 0), (unsigned long long)(v ? v[JV_BULK] : 0),
           (unsigned long long)(v ? v[JV_TENSOR] : 0), (unsigned long long)(v ? v[JV_CPASYNC] : 0),
           (unsigned long long)(ctx ? ctx->n_l2_groups : 0), last.c_str());
  std::string s = b;
  if (buf && cap) {
    size_t k = std::min(cap - 1, s.size());
    memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return (int64_t)s.size();
}

void* qs_get_stream(const qs_ctx* ctx, int i) {
  if (!ctx || i < 0 || i >= (int)ctx->shards.size()) return nullptr;
  return (void*)ctx->shards[i].stream;
}

int qs_set_timing(qs_ctx* ctx, int enable) {
  if (!ctx) return QS_EINVAL;
  {
    const int rc = finish_inflight(ctx);
    if (rc) return rc;
  }
  ctx->timing = enable != 0;
  ctx->accumulate = enable == 2;
  memset(ctx->k_count, 0, sizeof ctx->k_count);
  memset(ctx->k_ms, 0, sizeof ctx->k_ms);
  memset(ctx->k_bytes, 0, sizeof ctx->k_bytes);
  ctx->stats.t_device_ms = 0;
  ctx->stats.t_plan_ms = 0;
  ctx->launches = 0;
  return QS_OK;
}

int qs_get_kernel_timing(const qs_ctx* ctx, int kind, uint64_t* launches, double* ms,
                         uint64_t* bytes) {
  if (!ctx || kind < 0 || kind >= KK_NUM) return QS_EINVAL;
  {
    const int rc = finish_inflight(const_cast<qs_ctx*>(ctx));
    if (rc) return rc;
  }
  if (launches) *launches = ctx->k_count[kind];
  if (ms) *ms = ctx->k_ms[kind];
  if (bytes) *bytes = ctx->k_bytes[kind];
  return QS_OK;
}

}  // extern "C"
