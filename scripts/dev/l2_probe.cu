// f2 feasibility probe ("within the cache capacity"):
// how fast is one read+write "pass" over a buffer that stays resident in the
// 126 MB L2, and what does a grid-wide barrier between passes cost?
//
// (1) launch-per-pass: an in-place complex128 phase multiply (32 B/amp, the
//     K1 traffic shape) over S bytes, one launch per pass, S from 4 MiB to 4 GiB.
// (2) persistent: one cooperative kernel doing R passes over S bytes with
//     grid.sync() between them (the f2 two-level scheme's inner loop).
// Prints one JSON line per measurement. Standalone dev tool, not product code.
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_probe l2_probe.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ void rot(double2* a, size_t i, double c, double s) {
  double2 v = a[i];
  a[i] = make_double2(v.x * c - v.y * s, v.x * s + v.y * c);
}

__global__ void pass_kernel(double2* a, size_t n, double c, double s) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) rot(a, i, c, s);
}

// 4 independent 16 B loads in flight per thread before the stores (L2 latency hiding)
__global__ void pass_kernel_ilp4(double2* a, size_t n, double c, double s) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) v[k] = a[i + k * stride];
#pragma unroll
    for (int k = 0; k < 4; k++) a[i + k * stride] = make_double2(v[k].x * c - v[k].y * s, v[k].x * s + v[k].y * c);
  }
  for (; i < n; i += stride) rot(a, i, c, s);
}

__global__ void persistent_kernel(double2* a, size_t n, int reps, double c, double s) {
  cg::grid_group g = cg::this_grid();
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; r++) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) rot(a, i, c, s);
    g.sync();
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t max_bytes = 4ull << 30;
  double2* a;
  CK(cudaMalloc(&a, max_bytes));
  CK(cudaMemset(a, 0, max_bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double c = 0.6, s = 0.8;
  const size_t sizes_mib[] = {4, 8, 16, 24, 32, 48, 64, 80, 96, 128, 256, 1024, 4096};
  const int threads = 512;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, persistent_kernel, threads, 0));
  for (size_t mib : sizes_mib) {
    size_t bytes = mib << 20, n = bytes / 16;
    int grid = sms * per_sm;
    int reps = mib <= 128 ? 200 : (mib <= 1024 ? 20 : 5);
    // (1) one launch per pass
    for (int w = 0; w < 3; w++) pass_kernel<<<grid, threads>>>(a, n, c, s);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; r++) pass_kernel<<<grid, threads>>>(a, n, c, s);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double per = ms / reps;
    printf("{\"mode\":\"launch_per_pass\",\"MiB\":%zu,\"us_per_pass\":%.2f,\"GBps\":%.1f}\n", mib,
           per * 1e3, 2.0 * bytes / (per * 1e-3) / 1e9);
    // (1b) one launch per pass, 4 loads in flight per thread
    for (int w = 0; w < 3; w++) pass_kernel_ilp4<<<grid, threads>>>(a, n, c, s);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; r++) pass_kernel_ilp4<<<grid, threads>>>(a, n, c, s);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    per = ms / reps;
    printf("{\"mode\":\"launch_per_pass_ilp4\",\"MiB\":%zu,\"us_per_pass\":%.2f,\"GBps\":%.1f}\n", mib,
           per * 1e3, 2.0 * bytes / (per * 1e-3) / 1e9);
    // (2) persistent kernel, grid.sync between passes
    void* args[] = {&a, &n, &reps, (void*)&c, (void*)&s};
    for (int w = 0; w < 2; w++)
      CK(cudaLaunchCooperativeKernel((void*)persistent_kernel, grid, threads, args, 0, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    CK(cudaLaunchCooperativeKernel((void*)persistent_kernel, grid, threads, args, 0, 0));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    per = ms / reps;
    printf("{\"mode\":\"persistent_grid_sync\",\"MiB\":%zu,\"us_per_pass\":%.2f,\"GBps\":%.1f,\"grid\":%d}\n",
           mib, per * 1e3, 2.0 * bytes / (per * 1e-3) / 1e9, grid);
    fflush(stdout);
  }
  // barrier cost alone: persistent kernel over an empty buffer
  {
    size_t n = 0;
    int reps = 10000, grid = sms * per_sm;
    void* args[] = {&a, &n, &reps, (void*)&c, (void*)&s};
    CK(cudaLaunchCooperativeKernel((void*)persistent_kernel, grid, threads, args, 0, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    CK(cudaLaunchCooperativeKernel((void*)persistent_kernel, grid, threads, args, 0, 0));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("{\"mode\":\"grid_sync_only\",\"us_per_sync\":%.3f,\"grid\":%d}\n", ms * 1e3 / reps, grid);
  }
  CK(cudaFree(a));
  return 0;
}
