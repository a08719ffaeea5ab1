// tcgen05 GEMM / implicit-GEMM convolution for the bf16 plans (sm_100a).
//
//   D[M, N] = act(A[M, K] * W[N, K]^T + bias[N] + res[M, N])     (bf16 out)
//
// A is either a plain row-major activation matrix loaded by TMA (linear
// layers, 1x1/stride-1 convolutions) or the implicit im2col view of an NHWC
// activation gathered by four producer warps with zero-filling cp.async
// (k x k / strided convolutions; K ordered (r, s, c) to match OHWI weights).
// W (weights, K-major, K padded to 64) always arrives by TMA.  Both land in
// the canonical 128-byte-swizzled K-major layout the UMMA descriptors expect.
//
// Warp roles (persistent CTAs, one per SM, static round-robin tile order
// with N fastest so consecutive CTAs share the same A rows in L2):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5   epilogue: tcgen05.ld 32 lanes x 32 cols, +bias +res, act,
//               bf16 pack, 16-byte stores; TMEM double buffered (2 x BN cols)
//               so tile i's epilogue overlaps tile i+1's mainloop
//   warps 6-9   (gather mode) A producers, one output pixel (row) per thread
//
// Pipelines: smem full/empty ring (STAGES deep) between producers and the MMA
// thread; tmem full/empty pair between the MMA thread and the epilogue.
#include "common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;

template <int BN, bool GATHER>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BN * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (200 * 1024) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int THREADS = GATHER ? 320 : 192;
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64
                                   : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN, bool GATHER>
__global__ void __launch_bounds__(TcCfg<BN, GATHER>::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, const TcArgs a) {
  using Cfg = TcCfg<BN, GATHER>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ntiles = a.tiles_m * a.tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], GATHER ? 1 + 128 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    if (!GATHER) tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t / a.tiles_n) * TC_BM;
        const int n0 = (t % a.tiles_n) * BN;
        for (int kb = 0; kb < a.kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (GATHER) {
            mbar_arrive_expect_tx(&full[stage], Cfg::B_BYTES);
          } else {
            mbar_arrive_expect_tx(&full[stage], Cfg::A_BYTES + Cfg::B_BYTES);
            tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, &full[stage], kb * TC_BK, m0);
          }
          tma_load_2d(sB + stage * Cfg::B_BYTES, &tmB, &full[stage], kb * TC_BK, n0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(TC_BM, BN, 1u);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int as = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem_base + as * BN;
        for (int kb = 0; kb < a.kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(sA + stage * Cfg::A_BYTES));
          const uint64_t bd = smem_desc_sw128(smem_u32(sB + stage * Cfg::B_BYTES));
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            umma_bf16(dt, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[as]);
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3;
    int it = 0;
    const bool vec_ok = (a.ldo % 8 == 0) && (a.res == nullptr || a.ldres % 8 == 0);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int as = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int m0 = (t / a.tiles_n) * TC_BM;
      const int n0 = (t % a.tiles_n) * BN;
      mbar_wait(&tfull[as], aph);
      tc_fence_after();
      const int row = m0 + lg * 32 + lane;
      const uint32_t taddr = tmem_base + (uint32_t(lg * 32) << 16) + as * BN;
      constexpr int CH = BN >= 32 ? 32 : BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += CH) {
        float v[32];
        if constexpr (CH == 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        } else {
          uint32_t r[16];
          tmem_ld_32x32b_x16(taddr + c, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
        }
        const int col0 = n0 + c;
        if (row < a.M && col0 < a.N) {
          if (vec_ok && col0 + CH <= a.N) {
#pragma unroll
            for (int j = 0; j < CH; ++j) {
              if (a.bias) v[j] += __ldg(a.bias + col0 + j);
            }
            if (a.res) {
              const uint4* rp =
                  reinterpret_cast<const uint4*>(a.res + (size_t)row * a.ldres + col0);
#pragma unroll
              for (int q = 0; q < CH / 8; ++q) {
                uint4 u = __ldg(rp + q);
                uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  float2 f = unpack_bf16x2(w4[h]);
                  v[q * 8 + 2 * h] += f.x;
                  v[q * 8 + 2 * h + 1] += f.y;
                }
              }
            }
            uint4* op = reinterpret_cast<uint4*>(a.out + (size_t)row * a.ldo + col0);
#pragma unroll
            for (int q = 0; q < CH / 8; ++q) {
              uint4 u;
              u.x = pack_bf16x2(act_apply(v[q * 8 + 0], a.act), act_apply(v[q * 8 + 1], a.act));
              u.y = pack_bf16x2(act_apply(v[q * 8 + 2], a.act), act_apply(v[q * 8 + 3], a.act));
              u.z = pack_bf16x2(act_apply(v[q * 8 + 4], a.act), act_apply(v[q * 8 + 5], a.act));
              u.w = pack_bf16x2(act_apply(v[q * 8 + 6], a.act), act_apply(v[q * 8 + 7], a.act));
              op[q] = u;
            }
          } else {
            for (int j = 0; j < CH; ++j) {
              const int col = col0 + j;
              if (col >= a.N) break;
              float x = v[j];
              if (a.bias) x += a.bias[col];
              if (a.res) x += __bfloat162float(a.res[(size_t)row * a.ldres + col]);
              a.out[(size_t)row * a.ldo + col] = __float2bfloat16_rn(act_apply(x, a.act));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
    }
  } else if (GATHER) {
    // ------------------------------------------------------------ im2col gather
    constexpr int LAG = 2;
    const int g = threadIdx.x - 6 * 32;   // row of the A tile owned by this thread
    const uint32_t sw = g & 7;
    int stage = 0;
    uint32_t phase = 0;
    int issued = 0;
    const size_t img_elems = (size_t)a.H * a.W * a.C;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int m = (t / a.tiles_n) * TC_BM + g;
      const bool vrow = m < a.M;
      int img = 0, oh = 0, ow = 0;
      if (vrow) {
        img = m / a.OHW;
        const int rem = m - img * a.OHW;
        oh = rem / a.OW;
        ow = rem - oh * a.OW;
      }
      const int ih0 = oh * a.stride - a.pad;
      const int iw0 = ow * a.stride - a.pad;
      const bf16* xb = a.x + img * img_elems;
      for (int kb = 0; kb < a.kblocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t dst = smem_u32(sA + stage * Cfg::A_BYTES) + g * 128;
        if (a.c_div64) {
          // C % 64 == 0: the whole 64-wide K block is one filter tap
          const int k0 = kb * TC_BK;
          const int tap = k0 / a.C;
          const int c0 = k0 - tap * a.C;
          const int r = tap / a.S;
          const int s = tap - r * a.S;
          const int ih = ih0 + r, iw = iw0 + s;
          const bool ok = vrow && k0 < a.Kreal && (unsigned)ih < (unsigned)a.H &&
                          (unsigned)iw < (unsigned)a.W;
          const bf16* src = ok ? xb + ((size_t)ih * a.W + iw) * a.C + c0 : a.x;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            cp_async_16(dst + ((j ^ sw) << 4), ok ? src + j * 8 : a.x, ok ? 16u : 0u);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int k = kb * TC_BK + j * 8;
            const void* src = a.x;
            uint32_t bytes = 0;
            if (vrow && k < a.Kreal) {
              const int tap = k / a.C;
              const int c = k - tap * a.C;
              const int r = tap / a.S;
              const int s = tap - r * a.S;
              const int ih = ih0 + r, iw = iw0 + s;
              if ((unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W) {
                src = xb + ((size_t)ih * a.W + iw) * a.C + c;
                bytes = 16;
              }
            }
            cp_async_16(dst + ((j ^ sw) << 4), src, bytes);
          }
        }
        cp_async_commit();
        if (issued >= LAG) {
          cp_async_wait<LAG>();
          fence_proxy_async_smem();
          int ps = stage - LAG;
          if (ps < 0) ps += STAGES;
          mbar_arrive(&full[ps]);
        }
        ++issued;
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int i = (issued < LAG ? issued : LAG); i > 0; --i) {
      int ps = stage - i;
      if (ps < 0) ps += STAGES;
      mbar_arrive(&full[ps]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side

template <int BN, bool G>
static cudaError_t launch_bn(const TcArgs& a, const CUtensorMap& ta, const CUtensorMap& tb,
                             int num_sms, cudaStream_t st) {
  using Cfg = TcCfg<BN, G>;
  auto kern = tc_gemm_kernel<BN, G>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int tiles = a.tiles_m * a.tiles_n;
  const int grid = tiles < num_sms ? tiles : num_sms;
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(ta, tb, a);
  return cudaGetLastError();
}

int tc_pick_bn(long M, int N, int num_sms) {
  const int cands[5] = {256, 128, 64, 32, 16};
  long best_cost = -1;
  int best = 16;
  const long tm = (M + TC_BM - 1) / TC_BM;
  for (int bn : cands) {
    if (bn > 16 && bn / 2 >= N) continue;   // far wider than N: wasted columns
    const long tiles = tm * ((N + bn - 1) / bn);
    const long waves = (tiles + num_sms - 1) / num_sms;
    const long cost = waves * (bn > 128 ? bn : 128);   // MMA is smem-bound below N=128
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

cudaError_t tc_gemm_launch(const TcArgs& a, int bn, bool gather, const CUtensorMap& ta,
                           const CUtensorMap& tb, int num_sms, cudaStream_t st) {
#define B2_TC_CASE(BNV)                                                        \
  case BNV:                                                                    \
    return gather ? launch_bn<BNV, true>(a, ta, tb, num_sms, st)               \
                  : launch_bn<BNV, false>(a, ta, tb, num_sms, st);
  switch (bn) {
    B2_TC_CASE(16)
    B2_TC_CASE(32)
    B2_TC_CASE(64)
    B2_TC_CASE(128)
    B2_TC_CASE(256)
    default: return cudaErrorInvalidValue;
  }
#undef B2_TC_CASE
}

}  // namespace b2
