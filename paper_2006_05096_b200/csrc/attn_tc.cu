// Fused self-attention on tcgen05 for seq = 128, head_dim = 64 (BERT-base).
//
// One CTA (4 warps) per (sample, head):
//   1. TMA brings Q, K, V (each 128 x 64 bf16, 128B-swizzled) straight out of
//      the fused QKV activation [B*S, 3*H*64].
//   2. S = Q K^T on the tensor core (M=128 queries, N=128 keys, K=64) into TMEM.
//   3. Each thread owns one query row: tcgen05.ld its 128 scores, max /
//      exp2 / sum in registers, writes unnormalised P (bf16) into smem in the
//      K-major 128B-swizzled layout.
//   4. O = P V (M=128, N=64, K=128; V consumed MN-major as stored) into TMEM.
//   5. tcgen05.ld O, scale by 1/rowsum, 16-byte stores into ctx[B*S, H*64].
// Nothing but Q/K/V in and the context out touches HBM.
#include "common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int AT_S = 128, AT_D = 64;
constexpr int AT_SMEM = 3 * 16384 + 2 * 16384 + 1024 + 64;

// K-major A/B except B MN-major (bit 16) for the P*V product
__host__ __device__ constexpr uint32_t idesc_bmn(int M, int N) {
  return make_idesc(M, N, 1u) | (1u << 16);
}

B2_DEV uint64_t smem_desc_mn_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(8192 >> 4) << 16;   // LBO: next 64-element MN block (unused, N = 64)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO: next group of 8 K rows
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __launch_bounds__(128, 2)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, bf16* __restrict__ out, int H) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + 16384;
  uint8_t* sV = smem + 32768;
  uint8_t* sP = smem + 49152;   // two 16 KB atoms: keys 0-63, 64-127
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 81920);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);

  const int warp = warp_index_uniform(), lane = threadIdx.x & 31;
  const int b = blockIdx.x / H, h = blockIdx.x % H;
  const int row0 = b * AT_S;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = uniform_u32(*tslot);
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {   // converged warp, elected lane issues (common.cuh)
    if (elect_one()) {
      mbar_arrive_expect_tx(&bars[0], 3 * 16384);
      tma_load_2d(sQ, &tmQKV, &bars[0], h * AT_D, row0);
      tma_load_2d(sK, &tmQKV, &bars[0], (H + h) * AT_D, row0);
      tma_load_2d(sV, &tmQKV, &bars[0], (2 * H + h) * AT_D, row0);
    }
    __syncwarp();
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    const uint64_t dq = smem_desc_sw128(smem_u32(sQ));
    const uint64_t dk = smem_desc_sw128(smem_u32(sK));
#pragma unroll
    for (int k = 0; k < AT_D / 16; ++k)
      if (elect_one()) umma_bf16(tbase, dq + 2 * k, dk + 2 * k, make_idesc(128, 128, 1u), k ? 1u : 0u);
    if (elect_one()) umma_commit(&bars[1]);
  }
  mbar_wait(&bars[1], 0);
  tc_fence_after();

  // ---- softmax over this thread's query row (TMEM lane = row)
  const int row = warp * 32 + lane;
  const uint32_t trow = tbase + (uint32_t(warp * 32) << 16);
  float s[128];
  {
    uint32_t r[32];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      tmem_ld_32x32b_x32(trow + c * 32, r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) s[c * 32 + j] = __uint_as_float(r[j]);
    }
  }
  const float scl = 0.125f * 1.4426950408889634f;   // 1/sqrt(64) * log2(e)
  float mx = s[0];
#pragma unroll
  for (int j = 1; j < 128; ++j) mx = fmaxf(mx, s[j]);
  const float off = mx * scl;
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < 128; ++j) {
    s[j] = exp2f(fmaf(s[j], scl, -off));
    sum += s[j];
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {   // 8 keys per 16-byte chunk
    uint4 u;
    u.x = pack_bf16x2(s[8 * j + 0], s[8 * j + 1]);
    u.y = pack_bf16x2(s[8 * j + 2], s[8 * j + 3]);
    u.z = pack_bf16x2(s[8 * j + 4], s[8 * j + 5]);
    u.w = pack_bf16x2(s[8 * j + 6], s[8 * j + 7]);
    uint8_t* dst = sP + (j >> 3) * 16384 + row * 128 + ((((j & 7) ^ (row & 7))) << 4);
    *reinterpret_cast<uint4*>(dst) = u;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();

  if (warp == 0) {
    tc_fence_after();
    const uint32_t pbase = smem_u32(sP);
    const uint32_t vbase = smem_u32(sV);
#pragma unroll
    for (int k = 0; k < AT_S / 16; ++k) {
      const uint64_t da = smem_desc_sw128(pbase + (k >> 2) * 16384 + (k & 3) * 32);
      const uint64_t dv = smem_desc_mn_sw128(vbase + k * 16 * 128);
      if (elect_one()) umma_bf16(tbase + 128, da, dv, idesc_bmn(128, 64), k ? 1u : 0u);
    }
    if (elect_one()) umma_commit(&bars[1]);
  }
  mbar_wait(&bars[1], 1);
  tc_fence_after();

  const float inv = 1.f / sum;
  uint4* orow = reinterpret_cast<uint4*>(out + (size_t)(row0 + row) * (H * AT_D) + h * AT_D);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(trow + 128 + c * 32, r);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 u;
      u.x = pack_bf16x2(__uint_as_float(r[8 * q + 0]) * inv, __uint_as_float(r[8 * q + 1]) * inv);
      u.y = pack_bf16x2(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv);
      u.z = pack_bf16x2(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv);
      u.w = pack_bf16x2(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv);
      orow[c * 4 + q] = u;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

cudaError_t attention_tc(const CUtensorMap& tm_qkv, bf16* out, int B, int H, cudaStream_t st) {
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  return launch_pdl(attn_tc_kernel, dim3(B * H), dim3(128), AT_SMEM, st, tm_qkv, out, H);
}

}  // namespace b2
