// Fixed per-launch cost of persistent tcgen05 kernels: empty kernels with the
// GEMM's launch shape (148 x 320, 227 KB dynamic smem, TMEM alloc/dealloc,
// 5 tensor-map params), timed by events over 200 back-to-back launches.
#include <cstdio>
#include "common.cuh"
struct P5 { CUtensorMap m[5]; int x[64]; };
__global__ void k_empty(int) {}
__global__ void __launch_bounds__(320, 1) k_smem(int) { extern __shared__ uint8_t s[]; if (threadIdx.x == 999) s[0] = 1; }
__global__ void __launch_bounds__(320, 1) k_tmem(int) {
  extern __shared__ uint8_t s[];
  __shared__ uint32_t slot;
  if ((threadIdx.x >> 5) == 1) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if ((threadIdx.x >> 5) == 1) tmem_dealloc(slot, 512);
}
__global__ void __launch_bounds__(320, 1) k_params(const __grid_constant__ P5 p) {
  extern __shared__ uint8_t s[];
  if (threadIdx.x == 999) s[0] = (uint8_t)p.x[3];
}
template <typename F, typename A>
void timeit(const char* name, F f, A arg, int smem) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 10; ++i) f<<<148, 320, smem>>>(arg);
  cudaEventRecord(e0);
  for (int i = 0; i < 200; ++i) f<<<148, 320, smem>>>(arg);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-28s smem %6d: %.2f us/launch (%s)\n", name, smem, ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  P5 p{};
  timeit("empty", k_empty, 0, 0);
  timeit("empty", k_smem, 0, 0);
  timeit("227KB smem", k_smem, 0, 232448);
  timeit("227KB smem + tmem 512", k_tmem, 0, 232448);
  timeit("227KB smem + 5 tmaps", k_params, p, 232448);
  // graph of 50 launches
  cudaStream_t st; cudaStreamCreate(&st);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 50; ++i) k_tmem<<<148, 320, 232448, st>>>(0);
  cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, st); for (int r = 0; r < 4; ++r) cudaGraphLaunch(ge, st); cudaEventRecord(e1, st);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("graph, 227KB + tmem: %.2f us/launch\n", ms * 1e3 / 200);
}
