// Access-pattern roofline probe (dev tool, not part of the library): an
// in-place read+write pass over a 2^n complex128 state where each CTA
// iteration touches one "chunk" of 4096 amplitudes spread over 12 given bit
// positions -- the HBM access pattern of a K1 pass with those chunk
// positions, without its arithmetic or shared-memory exchanges.  Thread t
// holds 16 amplitudes: thread bits -> positions p[0..7], register bits ->
// p[8..11] (p[0..2] = 0,1,2 give 128 B coalesced runs, as in the kernels).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pattern_bw scripts/dev/pattern_bw.cu
//   /tmp/pattern_bw 30 0,1,2,3,4,5,6,7,8,9,10,11
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

typedef unsigned long long u64;

struct Pat {
  int pos[12];
  int nc[40];
  int n_nc;
};

__global__ void __launch_bounds__(256) pass(double2* __restrict__ s, Pat P, u64 n_chunks, double f) {
  const unsigned t = threadIdx.x;
  u64 toff = 0;
  for (int i = 0; i < 8; i++) toff |= (u64)((t >> i) & 1u) << P.pos[i];
  u64 roff[16];
#pragma unroll
  for (int r = 0; r < 16; r++) {
    u64 o = 0;
    for (int i = 0; i < 4; i++) o |= (u64)((r >> i) & 1) << P.pos[8 + i];
    roff[r] = o;
  }
  for (u64 c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    u64 base = 0;
    for (int i = 0; i < P.n_nc; i++) base |= ((c >> i) & 1ull) << P.nc[i];
    double2* p = s + (base | toff);
    double2 v[16];
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = p[roff[r]];
#pragma unroll
    for (int r = 0; r < 16; r++) p[roff[r]] = make_double2(v[r].x * f, v[r].y * f);
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 30;
  Pat P;
  memset(&P, 0, sizeof P);
  {
    const char* s = argc > 2 ? argv[2] : "0,1,2,3,4,5,6,7,8,9,10,11";
    int k = 0;
    for (const char* c = s; *c && k < 12;) {
      P.pos[k++] = atoi(c);
      while (*c && *c != ',') c++;
      if (*c == ',') c++;
    }
  }
  u64 cm = 0;
  for (int i = 0; i < 12; i++) cm |= 1ull << P.pos[i];
  for (int q = 0; q < n; q++)
    if (!(cm >> q & 1)) P.nc[P.n_nc++] = q;
  const u64 amps = 1ull << n, n_chunks = amps >> 12;
  double2* s;
  cudaMalloc(&s, amps * sizeof(double2));
  cudaMemset(s, 0, amps * sizeof(double2));
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int per : {2, 4, 8}) {
    const int grid = nsm * per;
    pass<<<grid, 256>>>(s, P, n_chunks, 1.0);
    cudaEventRecord(a);
    const int reps = 5;
    for (int i = 0; i < reps; i++) pass<<<grid, 256>>>(s, P, n_chunks, 1.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("{\"n\": %d, \"pos\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"gbs\": %.1f}\n", n,
           argc > 2 ? argv[2] : "0..11", per, ms, 2.0 * amps * 16 / (ms * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
