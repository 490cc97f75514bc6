// Microbenchmark: shared-memory atomic flavours on sm_100a (same-address vs spread addresses,
// POPC.INC (constant 1) vs ADD with a register operand, predicated/branchy vs dummy-redirected).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_atoms mb_atoms.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(unsigned* out, unsigned inc, int iters, unsigned spread) {
  __shared__ unsigned h[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned base = (w * 97u) & 2047u;
  unsigned x = lane * spread;
  for (int it = 0; it < iters; ++it) {
    const unsigned b = (base + x) & 2047u;
    if (MODE == 0) atomicAdd(&h[b], 1u);                      // POPC.INC
    if (MODE == 1) atomicAdd(&h[b], inc);                     // ATOMS.ADD register operand
    if (MODE == 2) atomicAdd(&h[b], (it & 7) == 0 ? 0x10001u : 1u);
    if (MODE == 3) {                                          // INC + redirected ADD (dummy slot when 0)
      atomicAdd(&h[b], 1u);
      const unsigned v = (it & 3) == 0 ? 0x10001u : 0u;
      atomicAdd(v ? &h[2048 + b] : &h[4064 + lane], v);
    }
    x += 7u * spread;
    base += 3u;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[5];
}

int main() {
  unsigned* out;
  cudaMalloc(&out, 4096 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (unsigned spread : {0u, 1u, 33u}) {
    for (int mode = 0; mode < 4; ++mode) {
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<148, 1024>>>(out, 1u, iters, spread);
        if (mode == 1) k<1><<<148, 1024>>>(out, 1u, iters, spread);
        if (mode == 2) k<2><<<148, 1024>>>(out, 1u, iters, spread);
        if (mode == 3) k<3><<<148, 1024>>>(out, 1u, iters, spread);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const double ops = 148.0 * 1024 * iters;
      printf("spread %2u mode %d: %.3f ms  %.2f atomic-steps/clk/SM (at 1.965 GHz)\n", spread, mode, best,
             ops / (best * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
