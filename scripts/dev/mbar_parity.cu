// mbarrier parity-wait semantics probe (bounded spins, no hangs)
#include <cstdio>
typedef unsigned long long u64;
__device__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ int tw(u64* b, unsigned par) {
  int ok = 0;
  for (int i = 0; i < 100000 && !ok; i++) {
    unsigned p;
    asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n selp.u32 %0, 1, 0, q;\n}"
                 : "=r"(p) : "r"(sa(b)), "r"(par) : "memory");
    ok = p;
  }
  return ok;
}
__global__ void k(int* out, const double* src) {
  __shared__ __align__(16) double buf[64];
  __shared__ u64 bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    out[0] = tw(&bar, 1);  // fresh, parity 1
    out[1] = tw(&bar, 0);  // fresh, parity 0 (expect 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 512;" :: "r"(sa(&bar)) : "memory");
    out[2] = tw(&bar, 1);  // after expect, before tx
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];"
                 :: "r"(sa(buf)), "l"(src), "r"(sa(&bar)) : "memory");
    out[3] = tw(&bar, 0);  // phase 0 done
    out[4] = tw(&bar, 1);  // parity 1 now = current phase 1 (expect 0)
  }
}
int main() {
  int* d; double* s;
  cudaMalloc(&d, 64); cudaMalloc(&s, 4096); cudaMemset(s, 0, 4096);
  k<<<1, 32>>>(d, s);
  int h[5];
  cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("err=%d fresh_p1=%d fresh_p0=%d after_expect_p1=%d done_p0=%d next_p1=%d\n", (int)e, h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
