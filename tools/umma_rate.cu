// Micro-benchmark: tcgen05.mma (kind::f16, cta_group::1, M = 128) issue
// throughput per SM as a function of N, A swizzle mode and A start-row offset
// (the shifted descriptors of conv_band.cu).  One CTA per SM, one converged
// warp issues `iters` MMAs back to back on resident shared-memory operands,
// then waits on a commit barrier; cycles per MMA from clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2006_05096_b200/csrc umma_rate.cu -o umma_rate
#include <cstdio>
#include <vector>
#include "common.cuh"

B2_DEV uint64_t desc_sw32(uint32_t a) {
  uint64_t d = (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;
  return d;
}

template <int N>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, int sw, int row_off, int nsteps,
                                                       long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = warp_index_uniform();
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = uniform_u32(slot);
  if (warp == 0) {
    constexpr uint32_t idesc = make_idesc(128, N, 1u);
    const uint32_t a0 = smem_u32(smem);
    const uint32_t b0 = smem_u32(smem + 96 * 1024);
    const uint32_t rb = sw == 128 ? 128 : 32;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // walk `nsteps` different shifted starts like conv_band's taps
      const int step = i % nsteps;
      const uint32_t aaddr = a0 + (uint32_t)(step * row_off) * rb;
      const uint64_t ad = sw == 128 ? smem_desc_sw128(aaddr) : desc_sw32(aaddr);
      const uint64_t bd = smem_desc_sw128(b0);
      if (elect_one()) umma_bf16(tbase + (i & 1) * N, ad, bd, idesc, 1u);
    }
    if (elect_one()) umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

template <int N>
void run(int sms, int sw, int row_off, int nsteps) {
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  const int iters = 4096;
  auto k = rate_kernel<N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  k<<<sms, 128, 170 * 1024>>>(iters, sw, row_off, nsteps, d);
  k<<<sms, 128, 170 * 1024>>>(iters, sw, row_off, nsteps, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(sms);
  cudaMemcpy(h.data(), d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (auto v : h) avg += v;
  avg /= sms;
  const double cyc = avg / iters;
  const double flop = 2.0 * 128 * N * 16;
  printf("N=%3d sw=%3d row_off=%3d nsteps=%d: %6.1f cyc/MMA  %7.1f FLOP/cyc/SM  (%s)\n", N, sw,
         row_off, nsteps, cyc, flop / cyc, cudaGetErrorString(e));
  cudaFree(d);
}


// CTA-pair variant: cluster of 2, the leader issues M = 256 (cta_group::2)
// MMAs; each CTA holds 128 rows of A and N/2 rows of B. Cycles per MMA on the
// leader -> per-SM FLOP/cycle = 2*128*N*16 / cyc (each SM computes 128 x N).
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    rate_pair_kernel(int iters, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = warp_index_uniform();
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  cluster_sync();
  if (warp == 0) tmem_alloc_pair(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = uniform_u32(slot);
  if (warp == 0 && rank == 0) {
    constexpr uint32_t idesc = make_idesc(256, N, 1u);
    const uint64_t ad = smem_desc_sw128(smem_u32(smem));
    const uint64_t bd = smem_desc_sw128(smem_u32(smem + 96 * 1024));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
      if (elect_one()) umma_bf16_pair(tbase + (i & 1) * N, ad, bd, idesc, 1u);
    if (elect_one()) umma_commit_pair(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  if (rank == 1 && warp == 0) mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, 512);
  }
}

template <int N>
void run_pair(int sms) {
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaMemset(d, 0, sms * sizeof(long long));
  const int iters = 4096;
  auto k = rate_pair_kernel<N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  k<<<sms, 128, 170 * 1024>>>(iters, d);
  k<<<sms, 128, 170 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(sms);
  cudaMemcpy(h.data(), d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  int n = 0;
  for (int i = 0; i < sms; i += 2) { avg += h[i]; ++n; }
  avg /= n;
  const double cyc = avg / iters;
  printf("PAIR M=256 N=%3d: %6.1f cyc/MMA  %7.1f FLOP/cyc/SM  (%s)\n", N, cyc,
         2.0 * 128 * N * 16 / cyc, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_pair<64>(sms - sms % 2);
  run_pair<128>(sms - sms % 2);
  run_pair<256>(sms - sms % 2);
  for (int off : {0, 8, 1, 3, 58}) {
    run<64>(sms, 128, off, off ? 9 : 1);
    run<128>(sms, 128, off, off ? 9 : 1);
    run<256>(sms, 128, off, off ? 9 : 1);
  }
  for (int off : {0, 8, 1, 115}) {
    run<64>(sms, 32, off, off ? 16 : 1);
    run<128>(sms, 32, off, off ? 16 : 1);
  }
  return 0;
}
