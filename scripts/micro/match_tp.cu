// Throughput of warp peer detection on B200: __match_any_sync vs ballots.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o match_tp match_tp.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE, int BITS>
__global__ void k(uint32_t *out, uint32_t seed, int iters) {
  uint32_t x = seed * (threadIdx.x + 1) * 2654435761u + blockIdx.x;
  uint32_t acc = 0;
  const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    uint32_t dg = (x >> 13) & ((1u << BITS) - 1u);
    if (MODE == 2) dg = 0;  // all lanes equal
    uint32_t peers;
    if (MODE == 0 || MODE == 2) {
      peers = __match_any_sync(0xffffffffu, dg);
    } else {
      peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < BITS; ++b) {
        const uint32_t B = __ballot_sync(0xffffffffu, (dg >> b) & 1u);
        peers &= ((dg >> b) & 1u) ? B : ~B;
      }
    }
    acc += __popc(peers & lt);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int BITS>
void run(const char *name) {
  uint32_t *o;
  cudaMalloc(&o, 148 * 8 * 1024 * 4);
  const int iters = 4096;
  k<MODE, BITS><<<148 * 2, 1024>>>(o, 1, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, BITS><<<148 * 2, 1024>>>(o, 1, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double warp_ops = 148.0 * 2 * 32 * iters;
  printf("%-28s bits=%d  %.3f ms  %.2f SM-cycles per warp-op (1.9 GHz)\n", name, BITS, ms,
         ms * 1e-3 * 1.9e9 * 148 / warp_ops);
  cudaFree(o);
}

int main() {
  run<0, 8>("match_any 8-bit digits");
  run<0, 4>("match_any 4-bit digits");
  run<0, 2>("match_any 2-bit digits");
  run<2, 8>("match_any all equal");
  run<1, 8>("ballots 8-bit digits");
  run<1, 4>("ballots 4-bit digits");
  return 0;
}
