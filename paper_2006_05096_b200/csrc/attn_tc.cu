// Fused self-attention on tcgen05 for seq = 128, head_dim = 64 (BERT-base).
//
// Per (sample, head) unit:
//   1. TMA brings Q, K, V (each 128 x 64 bf16, 128B-swizzled) straight out of
//      the fused QKV activation [B*S, 3*H*64].
//   2. S = Q K^T on the tensor core (M=128 queries, N=128 keys, K=64) into TMEM.
//   3. Each thread owns one query row: tcgen05.ld its 128 scores, padded
//      keys (attention-mask bits, when given) replaced by float32 min, max /
//      exp2 / sum in registers, writes unnormalised P (bf16) into smem in the
//      K-major 128B-swizzled layout.
//   4. O = P V (M=128, N=64, K=128; V consumed MN-major as stored) into TMEM.
//   5. tcgen05.ld O, scale by 1/rowsum, 16-byte stores into ctx[B*S, H*64].
// Nothing but Q/K/V in and the context out touches HBM.
#include "common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int AT_S = 128, AT_D = 64;

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

// Persistent, FOUR CTAs per SM walking (sample, head) units.  Each unit is a
// serial chain (load -> S MMA -> softmax -> P -> PV MMA -> context), so the
// SM is kept busy by several units in flight rather than by a pipeline inside
// one CTA: one CTA per SM ran 39 us per BERT layer at b=128, two (double-
// buffered, 99 KB, 256 TMEM columns each) 33 us.  Four fit because (a) P
// (128 x 128 bf16) overwrites the unit's Q|K region once S = QK^T is done and
// the CTA is single-buffered (48 KB), (b) O = PV is accumulated into the TMEM
// columns that held S (128 columns per CTA, 4 x 128 = the SM's 512), and (c)
// the softmax reads its 64 scores from TMEM twice in 32-column halves
// (max pass, then exp/sum/pack pass) so a thread holds 32 scores, not 64
// (<= 64 registers at 1024 threads per SM).  The next unit's Q/K/V load is
// issued as soon as PV has consumed P and V, overlapping the context stores.
// 8 warps: warps w and w + 4 share TMEM lane quadrant w & 3 (query rows) and
// split the 128 keys (and the 64 output columns) in halves; row max / sum are
// combined through shared memory.
constexpr int AT_WARPS = 8;
constexpr int AT_QKV = 3 * 16384;
constexpr int AT_SMEM = AT_QKV + 4 * 128 * 4 + 1024 + 64;
constexpr int AT_CTAS_PER_SM = 4;

// 2^x on the SFU alone (ex2.approx.ftz): exp2f adds a denormal-range rescue
// (compare, two conditional multiplies) that softmax arguments <= 0 never need
// beyond flushing results below 2^-126 to zero
B2_DEV float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

B2_DEV void at_bar() { asm volatile("bar.sync 1, %0;" ::"n"(AT_WARPS * 32) : "memory"); }

__global__ void __launch_bounds__(AT_WARPS * 32, AT_CTAS_PER_SM)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, bf16* __restrict__ out, int H,
                   int units, const uint32_t* __restrict__ keymask) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;                         // Q | K | V, 16 KB each
  uint8_t* sP = sQ;                           // two 16 KB atoms (keys 0-63, 64-127) over Q | K
  float* red = reinterpret_cast<float*>(smem + AT_QKV);   // [2 stats][2 halves][128 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 4 * 128);   // load, mma
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);

  const int warp = warp_index_uniform(), lane = threadIdx.x & 31;
  const int q = warp & 3, hh = warp >> 2;
  const int row = q * 32 + lane;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = uniform_u32(*tslot);
  pdl_wait();
  pdl_launch_dependents();

  auto issue_load = [&](int u) {
    const int b = u / H, h = u - (u / H) * H;
    mbar_arrive_expect_tx(&bars[0], AT_QKV);
    tma_load_2d(sQ, &tmQKV, &bars[0], h * AT_D, b * AT_S);
    tma_load_2d(sQ + 16384, &tmQKV, &bars[0], (H + h) * AT_D, b * AT_S);
    tma_load_2d(sQ + 32768, &tmQKV, &bars[0], (2 * H + h) * AT_D, b * AT_S);
  };
  if (threadIdx.x == 0 && (int)blockIdx.x < units) issue_load(blockIdx.x);

  const float scl = 0.125f * 1.4426950408889634f;   // 1/sqrt(64) * log2(e)
  uint32_t mph = 0;
  const uint32_t trow = tbase + (uint32_t(q * 32) << 16) + hh * 64;   // this thread's 64 scores
  int it = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
    // key-validity bits (attention mask) fetched before the waits: on the
    // critical path (after S) the L2 round trip was ~5% of the kernel's stalls
    uint32_t w0 = 0xffffffffu, w1 = 0xffffffffu;
    if (keymask) {
      const int bq = u / H;
      w0 = __ldg(keymask + bq * 4 + hh * 2);
      w1 = __ldg(keymask + bq * 4 + hh * 2 + 1);
    }
    mbar_wait(&bars[0], it & 1);
    __syncwarp();
    tc_fence_after();
    if (warp == 0) {   // S = Q K^T (M=128 queries, N=128 keys, K=64)
      const uint64_t dq = smem_desc_sw128(smem_u32(sQ));
      const uint64_t dk = smem_desc_sw128(smem_u32(sQ + 16384));
#pragma unroll
      for (int k = 0; k < AT_D / 16; ++k)
        if (elect_one()) umma_bf16(tbase, dq + 2 * k, dk + 2 * k, make_idesc(128, 128, 1u), k ? 1u : 0u);
      if (elect_one()) umma_commit(&bars[1]);
    }
    mbar_wait(&bars[1], mph);
    mph ^= 1;
    __syncwarp();
    tc_fence_after();

    // ---- softmax over this thread's row, key half hh (64 scores, two 32-column passes)
    float sv[32];
    auto load_half = [&](int half) {   // 32 scores; padded keys -> float32 min (exp2 underflows)
      uint32_t r[32];
      tmem_ld_32x32b_x32(trow + half * 32, r);
      tmem_wait_ld();
      const uint32_t w = half ? w1 : w0;
      if (w == 0xffffffffu) {   // no padded key in these 32 (warp-uniform: one sample, one half)
#pragma unroll
        for (int j = 0; j < 32; ++j) sv[j] = __uint_as_float(r[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          sv[j] = ((w >> j) & 1u) ? __uint_as_float(r[j]) : -3.4028234663852886e38f;
      }
    };
    float mx;
    load_half(0);
    mx = sv[0];
#pragma unroll
    for (int j = 1; j < 32; ++j) mx = fmaxf(mx, sv[j]);
    load_half(1);
#pragma unroll
    for (int j = 0; j < 32; ++j) mx = fmaxf(mx, sv[j]);
    red[hh * 128 + row] = mx;
    at_bar();
    mx = fmaxf(red[row], red[128 + row]);
    const float off = mx * scl;
    float sum = 0.f;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      load_half(half);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        sv[j] = ex2_ftz(fmaf(sv[j], scl, -off));
        sum += sv[j];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {   // 8 keys per 16-byte chunk of atom hh
        uint4 w;
        w.x = pack_bf16x2(sv[8 * j + 0], sv[8 * j + 1]);
        w.y = pack_bf16x2(sv[8 * j + 2], sv[8 * j + 3]);
        w.z = pack_bf16x2(sv[8 * j + 4], sv[8 * j + 5]);
        w.w = pack_bf16x2(sv[8 * j + 6], sv[8 * j + 7]);
        const int c16 = half * 4 + j;
        *reinterpret_cast<uint4*>(sP + hh * 16384 + row * 128 + ((c16 ^ (row & 7)) << 4)) = w;
      }
    }
    red[256 + hh * 128 + row] = sum;
    fence_proxy_async_smem();
    tc_fence_before();
    at_bar();
    sum = red[256 + row] + red[384 + row];

    if (warp == 0) {   // O = P V (M=128, N=64, K=128; V MN-major as stored) over S's columns
      tc_fence_after();
      const uint32_t pbase = smem_u32(sP);
      const uint32_t vbase = smem_u32(sQ + 32768);
#pragma unroll
      for (int k = 0; k < AT_S / 16; ++k) {
        const uint64_t da = smem_desc_sw128(pbase + (k >> 2) * 16384 + (k & 3) * 32);
        const uint64_t dv = smem_desc_mn_sw128(vbase + k * 16 * 128);
        if (elect_one()) umma_bf16(tbase, da, dv, idesc_bmn(128, 64), k ? 1u : 0u);
      }
      if (elect_one()) umma_commit(&bars[1]);
    }
    mbar_wait(&bars[1], mph);
    mph ^= 1;
    __syncwarp();
    tc_fence_after();
    // P and V consumed: the next unit's Q/K/V may land while we store the context
    if (threadIdx.x == 0 && u + (int)gridDim.x < units) issue_load(u + gridDim.x);

    // ---- context: this thread's row, output columns hh*32 .. +32
    const int b = u / H, h = u - (u / H) * H;
    const float inv = 1.f / sum;
    uint32_t r[32];
    tmem_ld_32x32b_x32(tbase + (uint32_t(q * 32) << 16) + hh * 32, r);
    tmem_wait_ld();
    uint4* orow = reinterpret_cast<uint4*>(out + (size_t)(b * AT_S + row) * (H * AT_D) + h * AT_D +
                                           hh * 32);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 w;
      w.x = pack_bf16x2(__uint_as_float(r[8 * j + 0]) * inv, __uint_as_float(r[8 * j + 1]) * inv);
      w.y = pack_bf16x2(__uint_as_float(r[8 * j + 2]) * inv, __uint_as_float(r[8 * j + 3]) * inv);
      w.z = pack_bf16x2(__uint_as_float(r[8 * j + 4]) * inv, __uint_as_float(r[8 * j + 5]) * inv);
      w.w = pack_bf16x2(__uint_as_float(r[8 * j + 6]) * inv, __uint_as_float(r[8 * j + 7]) * inv);
      orow[j] = w;
    }
    tc_fence_before();
    at_bar();   // O TMEM and the red[] stats are reused by the next unit
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 128);
  }
}

cudaError_t attention_tc(const CUtensorMap& tm_qkv, bf16* out, int B, int H,
                         const uint32_t* keymask, cudaStream_t st) {
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = B * H;
  const int slots = AT_CTAS_PER_SM * sms;
  return launch_pdl(attn_tc_kernel, dim3(units < slots ? units : slots), dim3(AT_WARPS * 32),
                    AT_SMEM, st, tm_qkv, out, H, units, keymask);
}

}  // namespace b2
