// Banded implicit-GEMM convolution on tcgen05 (sm_100a): stride-1 k x k
// convolutions whose A operand is loaded ONCE per band of output rows and
// reused by every filter tap through shifted shared-memory descriptors.
//
// The plain im2col path (gemm_tc.cu, a_im2col = 1) fetches a fresh 128 x 64
// A tile from L2 for every (tap, channel group): a 3x3 conv streams its input
// 9 times through the SM.  For the narrow-N layers (ResNet-50 layer1: N = 64)
// that A stream, not the MMA, bounds the kernel.  Here a work unit is a band
// of `bh` output rows of one image:
//
//   * one 4D TMA box loads the band's input rows plus halo, (bh + R - 1) rows x
//     Wp columns x CGW channels, with out-of-bounds (the conv padding) zero
//     filled by the TMA unit.  In shared memory the box is a matrix whose row
//     p = hh * Wp + ww is one input pixel (CGW channels, K-major, swizzled);
//   * output position p = oh * Wp + ow (band-local, padded-flattened) reads
//     tap (r, s) at row p + r * Wp + s, so the UMMA A operand of tap (r, s) for
//     M tile mt is the same matrix with its start address moved by
//     (mt * 128 + r * Wp + s) rows — no data movement per tap;
//   * positions with ow >= W (the Wp - W padding columns) or past the band are
//     computed and discarded by the epilogue (<= 12.5% for ResNet/VGG shapes).
//
// Two A layouts:
//   CGW = 64: 64-channel groups, 128-byte rows, SWIZZLE_128B (3x3 convs, C % 64 == 0)
//   CGW = 16: the 16-channel space-to-depth stem tensor, 32-byte rows, SWIZZLE_32B
// The swizzle is a function of the shared-memory address, so shifted starts
// that stay on row boundaries see the same pattern the TMA unit wrote.
//
// B (weights, K-major [N][Kpad], K order (r, s, c)) is either resident — all
// K blocks loaded once per CTA when they fit — or streamed per (tap, group)
// through a ring.  Accumulators: MT M tiles x BN fp32 columns in TMEM, double
// buffered so the epilogue of unit i overlaps the MMAs of unit i + 1.
//
// Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer,
// warps 2..9 epilogue (two per TMEM lane quadrant, splitting columns).
#include "common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int CB_EPI_WARPS = 8;
constexpr int CB_THREADS = (2 + CB_EPI_WARPS) * 32;
constexpr int CB_SMEM_MAX = 232448;
constexpr int CB_EPI_BYTES = CB_EPI_WARPS * 2 * 2048;   // per-warp double-buffered 32 x 64 B tiles

// SWIZZLE_32B K-major: rows of 32 B (16 bf16), 8-row atoms of 256 B
B2_DEV uint64_t smem_desc_sw32(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;             // LBO (unused: K extent is one atom)
  d |= (uint64_t)(256 >> 4) << 32;    // SBO: 8 rows x 32 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;             // SWIZZLE_32B
  return d;
}

// CGW = 8 (3-channel image inputs padded to 8): the band is a plain array of
// 16-byte pixels (no swizzle).  One K = 16 UMMA step covers TWO horizontally
// adjacent taps: in the non-swizzled K-major layout, core matrix 0 (K 0-7) is
// pixels p..p+7 and core matrix 1 (K 8-15) is pixels p+1..p+8, i.e. LBO = 16 B
// and SBO = 128 B over the same bytes.  Weights are laid out [N][r][4 taps][8]
// with the fourth tap zero, so a 3x3 conv is 6 UMMA steps per M tile.
template <int CGW>
B2_DEV uint64_t band_adesc(uint32_t addr) {
  if constexpr (CGW == 64) return smem_desc_sw128(addr);
  else if constexpr (CGW == 16) return smem_desc_sw32(addr);
  else return smem_desc_kmajor_noswizzle(addr, 16, 128);
}

// R x S taps and B residency are compile-time so the MMA issue loop unrolls
// to one descriptor add per operand per MMA: a single issuing thread has to
// keep up with 64-cycle (N <= 128) / 128-cycle (N = 256) MMAs, and a loop with
// runtime tap decomposition (integer division, parameter reloads) measured
// ~170 cycles per MMA — the tensor pipe then idles 80% of the time.
// CTA-local unit sequence: normally unit blockIdx.x + k * gridDim.x.  With
// the fused 2x2 pool on one-row bands (POOL, bh == 1) a CTA takes row PAIRS:
// its k-th unit is row (k & 1) of band pair blockIdx.x + (k >> 1) * gridDim.x,
// so the epilogue meets both rows of every pooled row (nbands is even).
template <bool POOL>
B2_DEV int band_unit(const BandArgs& a, int k, int units) {
  if (!POOL || a.bh != 1) {
    const long u = blockIdx.x + (long)k * gridDim.x;
    return u < units ? (int)u : -1;
  }
  const long pp = blockIdx.x + (long)(k >> 1) * gridDim.x;
  if (pp >= units / 2) return -1;
  const int nt = (int)(pp % a.tiles_n);
  long rest = pp / a.tiles_n;
  const int seg = (int)(rest % a.nseg);
  rest /= a.nseg;
  const int bp = (int)(rest % (a.nbands / 2));
  const int img = (int)(rest / (a.nbands / 2));
  const int band = 2 * bp + (k & 1);
  return ((img * a.nbands + band) * a.nseg + seg) * a.tiles_n + nt;
}

template <int BN, int CGW, int R, int S, bool BRES, int ACT, bool POOL = false>
__global__ void __launch_bounds__(CB_THREADS, 1)
    conv_band_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmO,
                     const __grid_constant__ CUtensorMap tmO2, const BandArgs a) {
  static_assert(!POOL || ACT == ACT_RELU || ACT == ACT_RELU6 || ACT == ACT_NONE,
                "the fused pool maxes before the activation: monotone activations only");
  constexpr int RB = CGW * 2;                 // bytes per A row (one pixel's channel group)
  constexpr int KSTEPS = CGW >= 16 ? CGW / 16 : 1;   // UMMA K steps per tap (CGW 8: per tap pair)
  constexpr int TAPS = R * S;
  constexpr int B_BLOCK = BN * 128;           // one 64-wide K block of weights
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + a.a_stages * a.a_stage_bytes;
  const int nb_bufs = BRES ? a.kblocks : a.b_stages;
  uint8_t* sEpi = sB + nb_bufs * B_BLOCK;     // 8 warps x 2 staging tiles of 32 x 64 B
  uint64_t* afull = reinterpret_cast<uint64_t*>(sEpi + CB_EPI_BYTES);
  uint64_t* aempty = afull + a.a_stages;
  uint64_t* bfull = aempty + a.a_stages;
  uint64_t* bempty = bfull + a.b_stages;
  uint64_t* tfull = bempty + a.b_stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = warp_index_uniform();
  const int lane = threadIdx.x & 31;
  const int units = a.B * a.nbands * a.nseg * a.tiles_n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.a_stages; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < a.b_stages; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], CB_EPI_WARPS);
    }
    mbar_init(bres, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmO);
    tma_prefetch_desc(&tmO2);
  }
  if (warp == 1) tmem_alloc(tmem_slot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = uniform_u32(*tmem_slot);
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // whole warp converged, one elected lane issues (see gemm_tc.cu)
    {
      const uint32_t afull_lo = uniform_u32(smem_u32(&afull[0]));
      const uint32_t aempty_lo = uniform_u32(smem_u32(&aempty[0]));
      const uint32_t bfull_lo = uniform_u32(smem_u32(&bfull[0]));
      const uint32_t bempty_lo = uniform_u32(smem_u32(&bempty[0]));
      const uint32_t sA_lo = uniform_u32(smem_u32(sA)), sB_lo = uniform_u32(smem_u32(sB));
      const uint32_t a_box = a.a_box_bytes, a_stage = a.a_stage_bytes;
      if constexpr (BRES) {
        if (elect_one()) {
          mbar_arrive_expect_tx(bres, (uint32_t)(a.kblocks * B_BLOCK));
          for (int kb = 0; kb < a.kblocks; ++kb)
            tma_load_2d(sB + kb * B_BLOCK, &tmB, bres, kb * 64, 0);
        }
        __syncwarp();
      }
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      for (int k = 0;; ++k) {
        const int u = band_unit<POOL>(a, k, units);
        if (u < 0) break;
        const int nt = u % a.tiles_n;
        const int rest = u / a.tiles_n;
        const int seg = rest % a.nseg;
        const int band = (rest / a.nseg) % a.nbands;
        const int img = rest / a.nseg / a.nbands;
        const int ax = seg * a.seg_w + a.x0, ay = band * a.bh + a.y0;
        for (int cg = 0; cg < a.CG; ++cg) {
          mbar_wait_u32(aempty_lo + as * 8, aph ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx_u32(afull_lo + as * 8, a_box);
            tma_load_4d_u32(sA_lo + as * a_stage, &tmA, afull_lo + as * 8, cg * CGW, ax, ay, img);
          }
          __syncwarp();
          if (++as == a.a_stages) {
            as = 0;
            aph ^= 1;
          }
          if constexpr (!BRES) {
            // one 64-wide K block per (tap, group): K index tap * C + cg * 64
#pragma unroll 1
            for (int t = 0; t < TAPS; ++t) {
              mbar_wait_u32(bempty_lo + bs * 8, bph ^ 1);
              if (elect_one()) {
                mbar_arrive_expect_tx_u32(bfull_lo + bs * 8, (uint32_t)B_BLOCK);
                tma_load_2d_u32(sB_lo + bs * B_BLOCK, &tmB, bfull_lo + bs * 8,
                                (t * a.CG + cg) * 64, nt * BN);
              }
              __syncwarp();
              if (++bs == a.b_stages) {
                bs = 0;
                bph ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // (whole warp, converged; one elected lane issues — see common.cuh)
    constexpr uint32_t idesc = make_idesc(128, BN, 1u);
    // per-tap A start offsets in descriptor units (16 B)
    uint32_t toff[TAPS];
#pragma unroll
    for (int t = 0; t < TAPS; ++t) toff[t] = (uint32_t)(((t / S) * a.Wp + (t % S)) * RB) >> 4;
    constexpr uint32_t MT_STEP = (128 * RB) >> 4;
    if constexpr (BRES) {
      mbar_wait(bres, 0);
      tc_fence_after();
    }
    const uint64_t bdesc0 = smem_desc_sw128(smem_u32(sB));
    int as = 0, bs = 0;
    uint32_t aph = 0, bph = 0;
    int it = 0;
    for (int k = 0;; ++k, ++it) {
      const int u = band_unit<POOL>(a, k, units);
      if (u < 0) break;
      const int seg = (u / a.tiles_n) % a.nseg;
      const int band = (u / a.tiles_n / a.nseg) % a.nbands;
      const int vr = min(a.bh, a.H - band * a.bh);
      const int segw = seg < a.nseg - 1 ? a.seg_w : a.W - seg * a.seg_w;
      const int mt_valid = ((vr - 1) * a.Wp + segw - 1) / 128 + 1;
      const int ab = it & 1;
      mbar_wait(&tempty[ab], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dbase = tmem_base + ab * a.MT * BN;
      if constexpr (BRES) {
        // CG == 1: K index of (tap t, step kk) = t * CGW + kk * 16
        mbar_wait(&afull[as], aph);
        tc_fence_after();
        const uint64_t adesc0 = band_adesc<CGW>(smem_u32(sA + as * a.a_stage_bytes));
        for (int mt = 0; mt < mt_valid; ++mt) {
          const uint64_t adm = adesc0 + mt * MT_STEP;
          if constexpr (CGW == 8) {
            // tap pairs (r, 2q) + (r, 2q + 1): A start = pixel r * Wp + 2q
#pragma unroll
            for (int r = 0; r < R; ++r) {
#pragma unroll
              for (int qq = 0; qq < (S + 1) / 2; ++qq) {
                const int kg = r * 32 + qq * 16;
                const uint32_t boff =
                    (uint32_t)((kg >> 6) * B_BLOCK + ((kg >> 4) & 3) * 32) >> 4;
                if (elect_one())
                  umma_bf16(dbase + mt * BN, adm + (uint32_t)(r * a.Wp + 2 * qq), bdesc0 + boff,
                            idesc, (r | qq) != 0 ? 1u : 0u);
              }
            }
            continue;
          }
#pragma unroll
          for (int t = 0; t < TAPS; ++t) {
#pragma unroll
            for (int kk = 0; kk < KSTEPS; ++kk) {
                const int kg = t * CGW + kk * 16;
              const uint32_t boff = (uint32_t)((kg >> 6) * B_BLOCK + ((kg >> 4) & 3) * 32) >> 4;
              if (elect_one())
                umma_bf16(dbase + mt * BN, adm + toff[t] + kk * 2, bdesc0 + boff, idesc,
                          (t | kk) != 0 ? 1u : 0u);
            }
          }
        }
        if (elect_one()) umma_commit(&aempty[as]);
        if (++as == a.a_stages) {
          as = 0;
          aph ^= 1;
        }
      } else {
        for (int cg = 0; cg < a.CG; ++cg) {
          mbar_wait(&afull[as], aph);
          tc_fence_after();
          const uint64_t adesc0 = band_adesc<CGW>(smem_u32(sA + as * a.a_stage_bytes));
#pragma unroll
          for (int t = 0; t < TAPS; ++t) {
            mbar_wait(&bfull[bs], bph);
            tc_fence_after();
            const uint64_t bd = bdesc0 + (uint32_t)((bs * B_BLOCK) >> 4);
            for (int mt = 0; mt < mt_valid; ++mt) {
#pragma unroll
              for (int kk = 0; kk < KSTEPS; ++kk)
                if (elect_one())
                  umma_bf16(dbase + mt * BN, adesc0 + mt * MT_STEP + toff[t] + kk * 2,
                            bd + kk * 2, idesc, (cg | t | kk) != 0 ? 1u : 0u);
            }
            if (elect_one()) umma_commit(&bempty[bs]);
            if (++bs == a.b_stages) {
              bs = 0;
              bph ^= 1;
            }
          }
          if (elect_one()) umma_commit(&aempty[as]);
          if (++as == a.a_stages) {
            as = 0;
            aph ^= 1;
          }
        }
      }
      if (elect_one()) umma_commit(&tfull[ab]);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // TMEM -> registers (+bias, act) -> bf16 -> 64B-swizzled 32 x 32 staging
    // tile -> TMA store.  The 4D output map [N, W, H, B] clips the padding
    // columns (ow >= W) in hardware; rows past the band's valid rows are
    // skipped so neighbouring bands are never overwritten.
    const int q = warp & 3;                 // TMEM lane quadrant
    const int ew = warp - 2;
    const int eh = ew >> 2;                 // column half
    uint8_t* obuf = sEpi + ew * 4096;
    uint32_t oi = 0;
    const uint32_t swz = (lane >> 1) & 3;
    float bpre[32];
    int bpre_n0 = -1;
    int it = 0;
    float prow[32];   // POOL, one-row bands: the pair's top row (raw accumulators)
    for (int k = 0;; ++k, ++it) {
      const int u = band_unit<POOL>(a, k, units);
      if (u < 0) break;
      const int nt = u % a.tiles_n;
      const int rest = u / a.tiles_n;
      const int seg = rest % a.nseg;
      const int band = (rest / a.nseg) % a.nbands;
      const int img = rest / a.nseg / a.nbands;
      const int vr = min(a.bh, a.H - band * a.bh);
      const int segw = seg < a.nseg - 1 ? a.seg_w : a.W - seg * a.seg_w;
      const int mt_valid = ((vr - 1) * a.Wp + segw - 1) / 128 + 1;
      const CUtensorMap* omap = seg == 0 ? &tmO : &tmO2;   // segment maps clip at their width
      const int n0 = nt * BN;
      const int ab = it & 1;
      if constexpr (BN == 64) {   // one 32-column chunk per warp: bias lives in registers
        if (n0 != bpre_n0) {
          const float4* bp = reinterpret_cast<const float4*>(a.bias + n0 + eh * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 b4 = __ldg(bp + j);
            bpre[4 * j] = b4.x;
            bpre[4 * j + 1] = b4.y;
            bpre[4 * j + 2] = b4.z;
            bpre[4 * j + 3] = b4.w;
          }
          bpre_n0 = n0;
        }
      }
      mbar_wait(&tfull[ab], (it >> 1) & 1);
      tc_fence_after();
      if constexpr (POOL) {
        // fused 2x2/2 max-pool (Wp == 128: M tile mt = band row mt; bh even):
        // rows 2j, 2j+1 meet in registers, column pairs across lanes 2i, 2i+1;
        // even lanes stage 16 pooled pixels x 32 channels, one TMA store
        const int segw0 = seg < a.nseg - 1 ? a.seg_w : a.W - seg * a.seg_w;
        if (a.bh == 1) {
          // rows meet across consecutive units (band_unit pairs them); BN = 64:
          // one 32-column chunk per warp
          const int p0 = q * 32;
          const int c = eh * 32;
          uint32_t ra[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + ab * a.MT * BN + c, ra);
          tmem_wait_ld();
          // max over the 2x2 window on the raw accumulators, then + bias and
          // the activation once: x -> act(x + b) is monotone (ReLU), so this
          // equals pooling the activated values
          float v[32];
          if ((k & 1) == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) prow[j] = __uint_as_float(ra[j]);
          } else if (n0 + c < a.N) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float m = fmaxf(__uint_as_float(ra[j]), prow[j]);
              v[j] = act_t<ACT>(fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1)) + bpre[j]);
            }
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            uint8_t* sbuf = obuf + (oi & 1) * 2048;
            if ((lane & 1) == 0) {
              const int pr = lane >> 1;
              const uint32_t pswz = (pr >> 1) & 3;
              uint8_t* orow = sbuf + pr * 64;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint4 w;
                w.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
                w.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
                w.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
                w.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
                *reinterpret_cast<uint4*>(orow + ((j ^ pswz) << 4)) = w;
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && p0 < segw0)
              tma_store_4d(omap, sbuf, n0 + c, p0 >> 1, band >> 1, img);
            if (lane == 0) bulk_commit();
            ++oi;
          }
        } else
        for (int mt = 0; mt + 1 < mt_valid; mt += 2) {
          const int r = mt;                              // band row of the pair's top
          if (r + 1 >= vr) break;
          const int p0 = q * 32;                         // column of lane 0 in the segment
#pragma unroll 1
          for (int c = eh * 32; c < BN && n0 + c < a.N; c += 64) {
            uint32_t ra[32], rb[32];
            const uint32_t tbase_mt =
                tmem_base + ((uint32_t)(q * 32) << 16) + ab * a.MT * BN + c;
            tmem_ld_32x32b_x32(tbase_mt + mt * BN, ra);
            tmem_ld_32x32b_x32(tbase_mt + (mt + 1) * BN, rb);
            float bv[32];
            if constexpr (BN == 64) {
#pragma unroll
              for (int j = 0; j < 32; ++j) bv[j] = bpre[j];
            } else {
              const float4* bp = reinterpret_cast<const float4*>(a.bias + n0 + c);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 b4 = __ldg(bp + j);
                bv[4 * j] = b4.x;
                bv[4 * j + 1] = b4.y;
                bv[4 * j + 2] = b4.z;
                bv[4 * j + 3] = b4.w;
              }
            }
            tmem_wait_ld();
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {   // pool the raw accumulators, then bias + act once
              const float m = fmaxf(__uint_as_float(ra[j]), __uint_as_float(rb[j]));
              v[j] = act_t<ACT>(fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1)) + bv[j]);
            }
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            uint8_t* sbuf = obuf + (oi & 1) * 2048;
            if ((lane & 1) == 0) {
              // 16 rows x 64 B, 64B-swizzled like the unpooled staging tile
              const int prow = lane >> 1;
              const uint32_t pswz = (prow >> 1) & 3;
              uint8_t* orow = sbuf + prow * 64;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                uint4 w;
                w.x = pack_bf16x2(v[8 * j + 0], v[8 * j + 1]);
                w.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
                w.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
                w.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
                *reinterpret_cast<uint4*>(orow + ((j ^ pswz) << 4)) = w;
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && p0 < segw0)
              tma_store_4d(omap, sbuf, n0 + c, p0 >> 1, (band * a.bh + r) >> 1, img);
            if (lane == 0) bulk_commit();
            ++oi;
          }
        }
      } else
      for (int mt = 0; mt < mt_valid; ++mt) {
        const int p0 = mt * 128 + q * 32;               // band position of lane 0
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + ab * a.MT * BN + mt * BN;
#pragma unroll 1
        for (int c = eh * 32; c < BN && n0 + c < a.N; c += 64) {   // columns >= N: nothing to store
          uint32_t rr[32];
          tmem_ld_32x32b_x32(taddr + c, rr);
          float bv[32];
          if constexpr (BN == 64) {
#pragma unroll
            for (int j = 0; j < 32; ++j) bv[j] = bpre[j];
          } else {
            const float4* bp = reinterpret_cast<const float4*>(a.bias + n0 + c);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 b4 = __ldg(bp + j);
              bv[4 * j] = b4.x;
              bv[4 * j + 1] = b4.y;
              bv[4 * j + 2] = b4.z;
              bv[4 * j + 3] = b4.w;
            }
          }
          tmem_wait_ld();
          if (lane == 0) bulk_wait_read<1>();          // staging buffer (oi & 1) free again
          __syncwarp();
          uint8_t* orow = obuf + (oi & 1) * 2048 + lane * 64;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float2 a2 = acc_add2(rr[8 * j + e], rr[8 * j + e + 1], bv[8 * j + e], bv[8 * j + e + 1]);
              w4[e / 2] = act_pack2<ACT>(a2.x, a2.y);
            }
            const uint4 w = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            *reinterpret_cast<uint4*>(orow + ((j ^ swz) << 4)) = w;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            // Wp is a multiple of 32 (a chunk lies in one output row; columns
            // >= W clip) or divides 32 (a chunk holds 32 / Wp whole rows; each
            // row's store starts at a 512 B-aligned staging offset).  TMA
            // stores reject negative coordinates, hence this geometry.
            const uint8_t* src = obuf + (oi & 1) * 2048;
            if (a.Wp >= 32) {
              const int r = p0 / a.Wp;
              if (r < vr) tma_store_4d(omap, src, n0 + c, p0 - r * a.Wp, band * a.bh + r, img);
            } else {
              for (int j = 0; j < 32 / a.Wp; ++j) {
                const int r = p0 / a.Wp + j;
                if (r < vr) tma_store_4d(omap, src + j * a.Wp * 64, n0 + c, 0, band * a.bh + r, img);
              }
            }
            bulk_commit();
          }
          ++oi;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// ------------------------------------------------------------------ CTA pair
// N = 64 convs with resident weights (ResNet layer1 3x3, VGG block 1) are
// capped by the ISA at half the tensor rate with M = 128 (a 128x64x16 UMMA
// takes as long as 128x128x16).  The pair form (cta_group::2, M = 256) at
// N = 64 measured 43 cycles per MMA instead of 2 x 64: 1.48x the per-SM rate
// (tools/umma_rate.cu).  Here the two CTAs of a cluster take bands u = 2p and
// 2p + 1 of the same unit order: each loads its own band box and half of the
// weight rows (32 of 64) into the same shared-memory offsets, the leader
// issues M = 256 UMMAs whose rows 0-127 come from its band and 128-255 from
// the peer's, and each CTA's epilogue drains its own TMEM lanes exactly as in
// conv_band_kernel.  An odd unit count leaves the last peer without a band:
// it re-loads the leader's band (the MMA needs both halves) and stores nothing.
template <int ACT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(CB_THREADS, 1)
    conv_band_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmO,
                          const __grid_constant__ CUtensorMap tmO2, const BandArgs a) {
  constexpr int BN = 64, RB = 128, R = 3, S = 3, TAPS = R * S, KSTEPS = 4;
  constexpr int B_BLOCK = (BN / 2) * 128;     // this CTA's 32 weight rows of one K block
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + a.a_stages * a.a_stage_bytes;
  uint8_t* sEpi = sB + a.kblocks * B_BLOCK;
  uint64_t* afull = reinterpret_cast<uint64_t*>(sEpi + CB_EPI_BYTES);
  uint64_t* aempty = afull + a.a_stages;
  uint64_t* tfull = aempty + a.a_stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = warp_index_uniform();
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int units = a.B * a.nbands * a.nseg;
  const int npairs = (units + 1) / 2;
  auto mtv = [&](int u) {
    const int seg = u % a.nseg;
    const int band = (u / a.nseg) % a.nbands;
    const int vr = min(a.bh, a.H - band * a.bh);
    const int segw = seg < a.nseg - 1 ? a.seg_w : a.W - seg * a.seg_w;
    return ((vr - 1) * a.Wp + segw - 1) / 128 + 1;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.a_stages; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * CB_EPI_WARPS);   // both CTAs' epilogue warps
    }
    mbar_init(bres, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmO);
    tma_prefetch_desc(&tmO2);
  }
  cluster_sync();                       // barrier inits visible to the peer
  if (warp == 1) tmem_alloc_pair(tmem_slot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = uniform_u32(*tmem_slot);
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      const uint32_t bres_l = mapa_shared(bres, 0);
      if (rank == 0) mbar_arrive_expect_tx(bres, (uint32_t)(2 * a.kblocks * B_BLOCK));
      for (int kb = 0; kb < a.kblocks; ++kb)
        tma_load_2d_pair(sB + kb * B_BLOCK, &tmB, bres_l, kb * 64, (int)rank * (BN / 2));
      int as = 0;
      uint32_t aph = 0;
      for (int p = cid; p < npairs; p += ncl) {
        int u = 2 * p + (int)rank;
        if (u >= units) u = 2 * p;                  // no band for the peer: reload the leader's
        const int seg = u % a.nseg;
        const int band = (u / a.nseg) % a.nbands;
        const int img = u / a.nseg / a.nbands;
        mbar_wait(&aempty[as], aph ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&afull[as], (uint32_t)(2 * a.a_box_bytes));
        tma_load_4d_pair(sA + as * a.a_stage_bytes, &tmA, mapa_shared(&afull[as], 0), 0,
                         seg * a.seg_w + a.x0, band * a.bh + a.y0, img);
        if (++as == a.a_stages) {
          as = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader, whole warp)
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc(256, BN, 1u);
      uint32_t toff[TAPS];
#pragma unroll
      for (int t = 0; t < TAPS; ++t) toff[t] = (uint32_t)(((t / S) * a.Wp + (t % S)) * RB) >> 4;
      constexpr uint32_t MT_STEP = (128 * RB) >> 4;
      mbar_wait(bres, 0);
      tc_fence_after();
      const uint64_t bdesc0 = smem_desc_sw128(smem_u32(sB));
      int as = 0;
      uint32_t aph = 0;
      int it = 0;
      for (int p = cid; p < npairs; p += ncl, ++it) {
        const int m0 = mtv(2 * p);
        const int m1 = 2 * p + 1 < units ? mtv(2 * p + 1) : m0;
        const int mt_valid = m0 > m1 ? m0 : m1;
        const int ab = it & 1;
        mbar_wait(&tempty[ab], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dbase = tmem_base + ab * a.MT * BN;
        mbar_wait(&afull[as], aph);
        tc_fence_after();
        const uint64_t adesc0 = smem_desc_sw128(smem_u32(sA + as * a.a_stage_bytes));
        for (int mt = 0; mt < mt_valid; ++mt) {
          const uint64_t adm = adesc0 + mt * MT_STEP;
#pragma unroll
          for (int t = 0; t < TAPS; ++t) {
#pragma unroll
            for (int kk = 0; kk < KSTEPS; ++kk) {
              const int kg = t * 64 + kk * 16;
              const uint32_t boff = (uint32_t)((kg >> 6) * B_BLOCK + ((kg >> 4) & 3) * 32) >> 4;
              if (elect_one())
                umma_bf16_pair(dbase + mt * BN, adm + toff[t] + kk * 2, bdesc0 + boff, idesc,
                               (t | kk) != 0 ? 1u : 0u);
            }
          }
        }
        if (elect_one()) umma_commit_pair(&aempty[as]);
        if (++as == a.a_stages) {
          as = 0;
          aph ^= 1;
        }
        if (elect_one()) umma_commit_pair(&tfull[ab]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    const int ew = warp - 2;
    const int eh = ew >> 2;
    uint8_t* obuf = sEpi + ew * 4096;
    uint32_t oi = 0;
    const uint32_t swz = (lane >> 1) & 3;
    const uint32_t trem = rank == 0 ? 0u : mapa_shared(&tempty[0], 0);
    float bpre[32];
    {
      const float4* bp = reinterpret_cast<const float4*>(a.bias + eh * 32);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 b4 = __ldg(bp + j);
        bpre[4 * j] = b4.x;
        bpre[4 * j + 1] = b4.y;
        bpre[4 * j + 2] = b4.z;
        bpre[4 * j + 3] = b4.w;
      }
    }
    int it = 0;
    for (int p = cid; p < npairs; p += ncl, ++it) {
      const int u = 2 * p + (int)rank;
      const int ab = it & 1;
      mbar_wait(&tfull[ab], (it >> 1) & 1);
      tc_fence_after();
      if (u < units) {
        const int seg = u % a.nseg;
        const int band = (u / a.nseg) % a.nbands;
        const int img = u / a.nseg / a.nbands;
        const int vr = min(a.bh, a.H - band * a.bh);
        const int mt_valid = mtv(u);
        const CUtensorMap* omap = seg == 0 ? &tmO : &tmO2;
        for (int mt = 0; mt < mt_valid; ++mt) {
          const int p0 = mt * 128 + q * 32;
          const uint32_t taddr =
              tmem_base + ((uint32_t)(q * 32) << 16) + ab * a.MT * BN + mt * BN + eh * 32;
          uint32_t rr[32];
          tmem_ld_32x32b_x32(taddr, rr);
          tmem_wait_ld();
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          uint8_t* orow = obuf + (oi & 1) * 2048 + lane * 64;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float2 a2 =
                  acc_add2(rr[8 * j + e], rr[8 * j + e + 1], bpre[8 * j + e], bpre[8 * j + e + 1]);
              w4[e / 2] = act_pack2<ACT>(a2.x, a2.y);
            }
            const uint4 w = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            *reinterpret_cast<uint4*>(orow + ((j ^ swz) << 4)) = w;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const uint8_t* src = obuf + (oi & 1) * 2048;
            if (a.Wp >= 32) {
              const int r = p0 / a.Wp;
              if (r < vr) tma_store_4d(omap, src, eh * 32, p0 - r * a.Wp, band * a.bh + r, img);
            } else {
              for (int j = 0; j < 32 / a.Wp; ++j) {
                const int r = p0 / a.Wp + j;
                if (r < vr) tma_store_4d(omap, src + j * a.Wp * 64, eh * 32, 0, band * a.bh + r, img);
              }
            }
            bulk_commit();
          }
          ++oi;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&tempty[ab]);
        else mbar_arrive_cluster(trem + ab * 8);
      }
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();                       // the peer's remote arrivals / the leader's MMAs are done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, a.tmem_cols);
  }
}

// ------------------------------------------------------------------ host side

int band_smem_bytes(const BandArgs& a, int bn) {
  const int nb = a.b_resident ? a.kblocks : a.b_stages;
  if (a.pair) bn /= 2;   // each CTA of a pair holds half the weight rows
  return 1024 + a.a_stages * a.a_stage_bytes + nb * bn * 128 + CB_EPI_BYTES +
         8 * (2 * a.a_stages + 2 * a.b_stages + 5) + 16;
}

// Fill the A-stage geometry of `a` for a band of `bh` rows.
static void band_geometry(BandArgs& a, int bh, int bn, int rb) {
  a.bh = bh;
  a.nbands = (a.H + bh - 1) / bh;
  a.MT = ((bh - 1) * a.Wp + a.seg_w - 1) / 128 + 1;
  const int box_rows = (bh + a.R - 1) * a.Wp;
  const int need_rows = a.MT * 128 + (a.R - 1) * a.Wp + (a.S - 1) + (rb == 16 ? 1 : 0);
  const int rows = ((box_rows > need_rows ? box_rows : need_rows) + 7) / 8 * 8;
  a.a_box_bytes = box_rows * rb;
  a.a_stage_bytes = (rows * rb + 1023) / 1024 * 1024;
  const int tmem = 2 * a.MT * bn;
  a.tmem_cols = tmem <= 32 ? 32 : tmem <= 64 ? 64 : tmem <= 128 ? 128 : tmem <= 256 ? 256 : 512;
}

// Choose band height (M tiles per band), pipeline depths and B residency.
// Candidates are ranked by the fraction of computed positions that are real
// outputs, then by B residency (no per-unit weight traffic), then by band
// size (less halo re-read).  Returns false when nothing fits (the caller
// keeps the im2col path).
bool band_config(BandArgs& a, int bn, int cgw, int mt_cap) {
  const int rb = cgw * 2;
  const int max_mt = 512 / (2 * bn);          // double-buffered accumulators in 512 TMEM cols
  if (max_mt < 1 || a.Wp > 256) return false;
  struct Cand { int bh, res, ast, bst; double eff; };
  Cand best{0, 0, 0, 0, 0.0};
  for (int mt = 1; mt <= max_mt && mt <= mt_cap; ++mt) {
    int bh = (mt * 128) / a.Wp;
    if (bh < 1) continue;
    if (bh > a.H) bh = a.H;
    if (a.pool2 && bh > 1 && (bh & 1)) continue;   // fused 2x2 pool: row pairs in or across bands
    const int bands = (a.H + bh - 1) / bh;
    double computed = 0.0;
    for (int b = 0; b < bands; ++b) {
      const int vr = (a.H - b * bh) < bh ? (a.H - b * bh) : bh;
      computed += (double)(((vr - 1) * a.Wp + a.seg_w - 1) / 128 + 1) * 128 * a.nseg;
    }
    Cand c{bh, 0, 0, 0, (double)a.H * a.W / computed};
    BandArgs t = a;
    band_geometry(t, bh, bn, rb);
    if (t.MT * 2 * bn > 512) continue;
    t.b_resident = 1;
    t.b_stages = 0;
    t.a_stages = 2;
    const bool res_ok = a.tiles_n == 1 && a.CG == 1 && bn == 64;   // instantiated resident kernels
    (void)0;
    if (res_ok && band_smem_bytes(t, bn) <= CB_SMEM_MAX) {
      c.res = 1;
      c.ast = (a.CG > 1 && (t.a_stages = 3, band_smem_bytes(t, bn) <= CB_SMEM_MAX)) ? 3 : 2;
    } else if (cgw == 64) {   // streamed B needs one (tap, group) per K block
      t.b_resident = 0;
      for (int ast = 3; ast >= 2 && !c.ast; --ast)
        for (int bst = 6; bst >= 3 && !c.ast; --bst) {
          t.a_stages = ast;
          t.b_stages = bst;
          if (band_smem_bytes(t, bn) <= CB_SMEM_MAX) {
            c.ast = ast;
            c.bst = bst;
          }
        }
    }
    if (!c.ast) continue;
    const bool better = !best.bh || c.eff > best.eff + 0.02 ||
                        (c.eff > best.eff - 0.02 && (c.res > best.res ||
                                                     (c.res == best.res && c.bh > best.bh)));
    if (better) best = c;
  }
  if (!best.bh) return false;
  band_geometry(a, best.bh, bn, rb);
  a.b_resident = best.res;
  a.a_stages = best.ast;
  a.b_stages = best.bst;
  return band_smem_bytes(a, bn) <= CB_SMEM_MAX;
}

template <int BN, int CGW, int R, int S, bool BRES, int ACT, bool POOL = false>
static cudaError_t band_launch_t(const BandArgs& a, const CUtensorMap& ta, const CUtensorMap& tb,
                                 const CUtensorMap& to, const CUtensorMap& to2, int num_sms,
                                 cudaStream_t st) {
  auto kern = conv_band_kernel<BN, CGW, R, S, BRES, ACT, POOL>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         CB_SMEM_MAX);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int units = a.B * a.nbands * a.nseg * a.tiles_n;
  const int grid = units < num_sms ? units : num_sms;
  return launch_pdl(kern, dim3(grid), dim3(CB_THREADS), band_smem_bytes(a, BN), st, ta, tb, to, to2,
                    a);
}

template <int ACT>
static cudaError_t band_pair_launch_t(const BandArgs& a, const CUtensorMap& ta,
                                      const CUtensorMap& tb, const CUtensorMap& to,
                                      const CUtensorMap& to2, int num_sms, cudaStream_t st) {
  auto kern = conv_band_pair_kernel<ACT>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         CB_SMEM_MAX);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int npairs = (a.B * a.nbands * a.nseg + 1) / 2;
  const int pairs = npairs < num_sms / 2 ? npairs : num_sms / 2;
  return launch_pdl(kern, dim3(2 * pairs), dim3(CB_THREADS), band_smem_bytes(a, 64), st, ta, tb,
                    to, to2, a);
}

template <int ACT>
static cudaError_t band_dispatch(const BandArgs& a, int bn, int cgw, const CUtensorMap& ta,
                                 const CUtensorMap& tb, const CUtensorMap& to,
                                 const CUtensorMap& to2, int num_sms, cudaStream_t st) {
  if (cgw == 16) {   // space-to-depth stems: 7x7/2 -> 4 x 4 taps, 3x3/2 -> 2 x 4
    if (bn == 64 && a.R == 4 && a.S == 4 && a.b_resident && a.CG == 1)
      return band_launch_t<64, 16, 4, 4, true, ACT>(a, ta, tb, to, to2, num_sms, st);
    if (bn == 64 && a.R == 2 && a.S == 4 && a.b_resident && a.CG == 1)
      return band_launch_t<64, 16, 2, 4, true, ACT>(a, ta, tb, to, to2, num_sms, st);
    return cudaErrorInvalidValue;
  }
  if (cgw == 8) {    // 3x3 on an 8-channel padded image (VGG conv1_1)
    if (bn == 64 && a.R == 3 && a.S == 3 && a.b_resident && a.CG == 1)
      return band_launch_t<64, 8, 3, 3, true, ACT>(a, ta, tb, to, to2, num_sms, st);
    return cudaErrorInvalidValue;
  }
  if (a.R != 3 || a.S != 3) return cudaErrorInvalidValue;
  if (a.pair) {
    if (bn == 64 && a.CG == 1 && a.b_resident && a.tiles_n == 1)
      return band_pair_launch_t<ACT>(a, ta, tb, to, to2, num_sms, st);
    return cudaErrorInvalidValue;
  }
  if (a.pool2) {   // fused 2x2 max-pool (VGG): ReLU only (checked on the host)
    if constexpr (ACT == ACT_RELU) {
      if (bn == 64 && a.b_resident && a.CG == 1 && a.bh == 1)
        return band_launch_t<64, 64, 3, 3, true, ACT_RELU, true>(a, ta, tb, to, to2, num_sms, st);
      if (bn == 128 && !a.b_resident)
        return band_launch_t<128, 64, 3, 3, false, ACT_RELU, true>(a, ta, tb, to, to2, num_sms, st);
    }
    return cudaErrorInvalidValue;
  }
  if (a.b_resident) {
    if (bn == 64 && a.CG == 1) return band_launch_t<64, 64, 3, 3, true, ACT>(a, ta, tb, to, to2, num_sms, st);
    return cudaErrorInvalidValue;
  }
  switch (bn) {
    case 64: return band_launch_t<64, 64, 3, 3, false, ACT>(a, ta, tb, to, to2, num_sms, st);
    case 128: return band_launch_t<128, 64, 3, 3, false, ACT>(a, ta, tb, to, to2, num_sms, st);
    case 256: return band_launch_t<256, 64, 3, 3, false, ACT>(a, ta, tb, to, to2, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

// Which (taps, BN, residency) combinations have a kernel instance.
bool band_supported(const BandArgs& a, int bn, int cgw, int act) {
  if (act != ACT_NONE && act != ACT_RELU && !(act == ACT_RELU6 && cgw == 16)) return false;
  if (cgw == 16)
    return bn == 64 && (a.R == 4 || a.R == 2) && a.S == 4 && a.b_resident && a.CG == 1 &&
           (act != ACT_RELU6 || a.R == 2);
  if (cgw == 8) return bn == 64 && a.R == 3 && a.S == 3 && a.b_resident && a.CG == 1;
  if (a.R != 3 || a.S != 3) return false;
  if (a.b_resident) return bn == 64 && a.CG == 1;
  return bn == 64 || bn == 128 || bn == 256;
}

cudaError_t conv_band_launch(const BandArgs& a, int bn, int cgw, const CUtensorMap& ta,
                             const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& to2,
                             int num_sms, cudaStream_t st) {
  if (a.act == ACT_RELU) return band_dispatch<ACT_RELU>(a, bn, cgw, ta, tb, to, to2, num_sms, st);
  if (a.act == ACT_NONE) return band_dispatch<ACT_NONE>(a, bn, cgw, ta, tb, to, to2, num_sms, st);
  if (a.act == ACT_RELU6 && cgw == 16 && bn == 64 && a.R == 2 && a.S == 4 && a.b_resident)
    return band_launch_t<64, 16, 2, 4, true, ACT_RELU6>(a, ta, tb, to, to2, num_sms, st);
  return cudaErrorInvalidValue;
}

// ============================================================================
// Stem convolution fused with its 3x3 / stride-2 / pad-1 max-pool.
//
// The space-to-depth stem (CGW = 16, 4 x 4 taps, Wp = 128: one conv output
// row per M tile) is computed two conv rows at a time — the rows 2ph, 2ph+1
// of pooled row ph — and never written to HBM.  The epilogue drops ReLU'd
// bf16 conv rows into a 3-slot shared-memory ring (slot = conv row mod 3,
// columns -1 and OW zero), then all epilogue threads max-pool pooled row ph
// from ring rows 2ph-1, 2ph, 2ph+1 and store it.  Zero stands in for the
// pool's -inf padding: every window holds at least one real, post-ReLU (>= 0)
// value, so the max is unchanged (requires ACT = ReLU; checked on the host).
//
// Each CTA owns a contiguous range of pooled rows so conv row 2ph-1 is still
// in the ring from the previous unit; only the first unit of a range that
// starts mid-image recomputes it (a third M tile).  Saves the 411 MB conv
// output write + re-read of the unfused stem/max-pool pair at ResNet b=256.
constexpr int SP_RING_SLOTS = 3;

B2_DEV void named_bar_epi() { asm volatile("bar.sync 1, %0;" ::"n"(CB_EPI_WARPS * 32) : "memory"); }

__global__ void __launch_bounds__(CB_THREADS, 1)
    stem_pool_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, const BandArgs a) {
  constexpr int BN = 64, CGW = 16, R = 4, S = 4, TAPS = 16, RB = 32, B_BLOCK = BN * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int ring_slot = (a.W + 2) * 128;          // (OW + 2) columns x 64 ch x bf16
  uint8_t* sA = smem;
  uint8_t* sB = sA + a.a_stages * a.a_stage_bytes;
  uint8_t* ring = sB + a.kblocks * B_BLOCK;
  uint64_t* afull = reinterpret_cast<uint64_t*>(ring + SP_RING_SLOTS * ring_slot);
  uint64_t* aempty = afull + a.a_stages;
  uint64_t* tfull = aempty + a.a_stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = warp_index_uniform();
  const int lane = threadIdx.x & 31;
  const int pairs = a.B * a.PH;                   // units: pooled rows of the whole batch
  const int u0 = (int)((long)blockIdx.x * pairs / gridDim.x);
  const int u1 = (int)((long)(blockIdx.x + 1) * pairs / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.a_stages; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], CB_EPI_WARPS);
    }
    mbar_init(bres, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, a.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = uniform_u32(*tmem_slot);
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_arrive_expect_tx(bres, (uint32_t)(a.kblocks * B_BLOCK));
      for (int kb = 0; kb < a.kblocks; ++kb) tma_load_2d(sB + kb * B_BLOCK, &tmB, bres, kb * 64, 0);
      int as = 0;
      uint32_t aph = 0;
      for (int u = u0; u < u1; ++u) {
        const int img = u / a.PH, ph = u - img * a.PH;
        const bool halo = u == u0 && ph > 0;
        mbar_wait(&aempty[as], aph ^ 1);
        mbar_arrive_expect_tx(&afull[as], (uint32_t)a.a_box_bytes);
        tma_load_4d(sA + as * a.a_stage_bytes, &tmA, &afull[as], 0, 0, 2 * ph - (halo ? 1 : 0), img);
        if (++as == a.a_stages) {
          as = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc(128, BN, 1u);
    uint32_t toff[TAPS];
#pragma unroll
    for (int t = 0; t < TAPS; ++t) toff[t] = (uint32_t)(((t / S) * a.Wp + (t % S)) * RB) >> 4;
    const uint32_t mt_step = (uint32_t)(a.Wp * RB) >> 4;   // one conv row = one s2d row
    mbar_wait(bres, 0);
    tc_fence_after();
    const uint64_t bdesc0 = smem_desc_sw128(smem_u32(sB));
    int as = 0;
    uint32_t aph = 0;
    int it = 0;
    for (int u = u0; u < u1; ++u, ++it) {
      const int ph = u % a.PH;
      const int nt = (u == u0 && ph > 0) ? 3 : 2;
      const int ab = it & 1;
      mbar_wait(&tempty[ab], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dbase = tmem_base + ab * 3 * BN;
      mbar_wait(&afull[as], aph);
      tc_fence_after();
      const uint64_t adesc0 = smem_desc_sw32(smem_u32(sA + as * a.a_stage_bytes));
      for (int mt = 0; mt < nt; ++mt) {
#pragma unroll
        for (int t = 0; t < TAPS; ++t) {
          const int kg = t * CGW;
          const uint32_t boff = (uint32_t)((kg >> 6) * B_BLOCK + ((kg >> 4) & 3) * 32) >> 4;
          if (elect_one())
            umma_bf16(dbase + mt * BN, adesc0 + mt * mt_step + toff[t], bdesc0 + boff, idesc,
                      t != 0 ? 1u : 0u);
        }
      }
      if (elect_one()) umma_commit(&aempty[as]);
      if (++as == a.a_stages) {
        as = 0;
        aph ^= 1;
      }
      if (elect_one()) umma_commit(&tfull[ab]);
    }
  } else {
    // ------------------------------------------------------------ epilogue + pool
    const int et = threadIdx.x - 64;                 // 0..255
    const int q = warp & 3;
    const int eh = (warp - 2) >> 2;
    for (int i = et; i < SP_RING_SLOTS * ring_slot / 16; i += CB_EPI_WARPS * 32)
      reinterpret_cast<uint4*>(ring)[i] = make_uint4(0, 0, 0, 0);
    float bv[32];
    {
      const float4* bp = reinterpret_cast<const float4*>(a.bias + eh * 32);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 b4 = __ldg(bp + j);
        bv[4 * j] = b4.x;
        bv[4 * j + 1] = b4.y;
        bv[4 * j + 2] = b4.z;
        bv[4 * j + 3] = b4.w;
      }
    }
    named_bar_epi();
    const int ow = q * 32 + lane;                    // this thread's conv column
    const int cidx = ow + 1;                         // ring column (0 and W+1 stay zero)
    int it = 0;
    for (int u = u0; u < u1; ++u, ++it) {
      const int img = u / a.PH, ph = u - img * a.PH;
      const bool halo = u == u0 && ph > 0;
      const int first = 2 * ph - (halo ? 1 : 0);
      const int nt = halo ? 3 : 2;
      const int ab = it & 1;
      mbar_wait(&tfull[ab], (it >> 1) & 1);
      tc_fence_after();
      for (int mt = 0; mt < nt; ++mt) {
        const int cr = first + mt;
        uint32_t rr[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + ab * 3 * BN + mt * BN + eh * 32, rr);
        tmem_wait_ld();
        if (ow < a.W) {
          uint8_t* col = ring + (cr % SP_RING_SLOTS) * ring_slot + cidx * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w4[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const float2 a2 = acc_add2(rr[8 * j + e], rr[8 * j + e + 1], bv[8 * j + e], bv[8 * j + e + 1]);
              w4[e / 2] = act_pack2<ACT_RELU>(a2.x, a2.y);
            }
            const uint4 w = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            const int chunk = eh * 4 + j;
            *reinterpret_cast<uint4*>(col + ((chunk ^ (cidx & 7)) << 4)) = w;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);       // accumulators free for unit it + 2
      if (ph == 0) {                                 // conv row -1 (pool padding): zeros
        uint8_t* slot = ring + ((SP_RING_SLOTS - 1) % SP_RING_SLOTS) * ring_slot;
        for (int i = et; i < ring_slot / 16; i += CB_EPI_WARPS * 32)
          reinterpret_cast<uint4*>(slot)[i] = make_uint4(0, 0, 0, 0);
      }
      named_bar_epi();
      // pooled row ph: max over conv rows 2ph-1..2ph+1, columns 2pw-1..2pw+1
      const uint8_t* r0 = ring + ((2 * ph + 2) % SP_RING_SLOTS) * ring_slot;
      const uint8_t* r1 = ring + ((2 * ph) % SP_RING_SLOTS) * ring_slot;
      const uint8_t* r2 = ring + ((2 * ph + 1) % SP_RING_SLOTS) * ring_slot;
      bf16* orow = a.pout + ((size_t)(img * a.PH + ph) * a.PW) * BN;
      for (int i = et; i < a.PW * 8; i += CB_EPI_WARPS * 32) {
        const int pw = i >> 3, v = i & 7;
        __nv_bfloat162 m[4];
        bool init = false;
#pragma unroll
        for (int dc = 0; dc < 3; ++dc) {
          const int c = 2 * pw + dc;                 // ring column of conv col 2pw-1+dc
          const int off = c * 128 + ((v ^ (c & 7)) << 4);
#pragma unroll
          for (int rr_ = 0; rr_ < 3; ++rr_) {
            const uint8_t* rp = rr_ == 0 ? r0 : rr_ == 1 ? r1 : r2;
            const uint4 x = *reinterpret_cast<const uint4*>(rp + off);
            const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
            for (int k = 0; k < 4; ++k) m[k] = init ? __hmax2(m[k], xh[k]) : xh[k];
            init = true;
          }
        }
        *reinterpret_cast<uint4*>(orow + pw * BN + v * 8) = *reinterpret_cast<const uint4*>(m);
      }
      named_bar_epi();                               // ring reads done before the next unit
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

static int stem_pool_smem(const BandArgs& a) {
  return 1024 + a.a_stages * a.a_stage_bytes + a.kblocks * 64 * 128 +
         SP_RING_SLOTS * (a.W + 2) * 128 + 8 * (2 * a.a_stages + 5) + 16;
}

// Geometry for the fused stem: box of 3 conv rows' worth of s2d rows (the
// halo unit), 3 M tiles per unit at most, resident weights.
bool stem_pool_config(BandArgs& a) {
  if (a.R != 4 || a.S != 4 || a.CG != 1 || a.N != 64 || a.Wp != 128 || a.W > 128 ||
      a.tiles_n != 1 || (a.H & 1) || (a.W & 1) || a.kblocks != 4)
    return false;
  a.MT = 3;
  a.bh = 2;
  const int box_rows = (3 + a.R - 1) * a.Wp;
  const int need_rows = 3 * 128 + (a.R - 1) * a.Wp + (a.S - 1);
  const int rows = ((box_rows > need_rows ? box_rows : need_rows) + 7) / 8 * 8;
  a.a_box_bytes = box_rows * 32;
  a.a_stage_bytes = (rows * 32 + 1023) / 1024 * 1024;
  a.tmem_cols = 512;
  a.b_resident = 1;
  a.b_stages = 0;
  for (a.a_stages = 4; a.a_stages >= 2; --a.a_stages)
    if (stem_pool_smem(a) <= CB_SMEM_MAX) return true;
  return false;
}

cudaError_t stem_pool_launch(const BandArgs& a, const CUtensorMap& ta, const CUtensorMap& tb,
                             int num_sms, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(stem_pool_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CB_SMEM_MAX);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int pairs = a.B * a.PH;
  const int grid = pairs < num_sms ? pairs : num_sms;
  return launch_pdl(stem_pool_kernel, dim3(grid), dim3(CB_THREADS), stem_pool_smem(a), st, ta, tb,
                    a);
}

}  // namespace b2
