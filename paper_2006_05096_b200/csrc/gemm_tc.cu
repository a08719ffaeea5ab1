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
//   warps 2-5   epilogue: tcgen05.ld (32 lanes x 64 cols per chunk), +bias,
//               +residual (prefetched one chunk ahead into registers), act,
//               bf16 pack into a 128B-swizzled staging tile, per-warp TMA
//               store; TMEM double buffered (2 x BN cols) so tile i's
//               epilogue overlaps tile i+1's mainloop
//   warps 6-9   (gather mode) A producers, one output pixel (row) per thread;
//               completion is signalled with cp.async.mbarrier.arrive so the
//               producers never wait on their own loads
//
// Pipelines: smem full/empty ring (a.stages deep, sized on the host from the
// 227 KB budget) between producers and the MMA thread; tmem full/empty pair
// between the MMA thread and the epilogue.
#include "common.cuh"
#include "kernels.h"

namespace b2 {

// Profiling aids (drain-only epilogues, phase timestamps) exist only in
// -DB2_DEBUG builds; production kernels carry no debug branches.
#ifdef B2_DEBUG
#define EPI_DBG(a) ((a).epi_debug)
#define TS_DBG(a) ((a).ts_debug)
#else
#define EPI_DBG(a) 0
#define TS_DBG(a) 0
#endif

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;
constexpr int TC_SMEM_MAX = 232448;           // 227 KB: the opt-in per-CTA maximum
constexpr int TC_EPI_WARPS = 8;               // two warps per TMEM lane quadrant
constexpr int TC_EPI_BYTES = TC_EPI_WARPS * 2 * 2048;   // 2 staging tiles of 32 x 64 B each
constexpr int TC_BAR_BYTES = 512;

template <int BN, bool GATHER>
struct TcCfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = BN * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int MAX_STAGES_RAW =
      (TC_SMEM_MAX - TC_EPI_BYTES - 1024 - TC_BAR_BYTES) / STAGE_BYTES;
  static constexpr int MAX_STAGES = MAX_STAGES_RAW > 8 ? 8 : MAX_STAGES_RAW;
  static constexpr int THREADS = (2 + TC_EPI_WARPS + (GATHER ? 4 : 0)) * 32;
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64
                                   : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM =
      MAX_STAGES * STAGE_BYTES + TC_EPI_BYTES + 1024 + TC_BAR_BYTES;
};

B2_DEV void add_bf16x8(float* v, const uint4& u) {
  const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int h = 0; h < 4; ++h) {   // packed add.rn.f32x2 (per-lane identical)
    const float2 f = unpack_bf16x2(w4[h]);
    f2unpack(f2add(f2pack(v[2 * h], v[2 * h + 1]), f2pack(f.x, f.y)), v[2 * h], v[2 * h + 1]);
  }
}

// TMA-store epilogue of one warp, specialised on the activation so the
// per-element math is branch-free.
// B2_GEMM_TS=2: per-tile stamps of CTA 0's first 32 tiles (globaltimer, ns):
// [0] producer past empty-wait, [1] MMA past full-wait, [2] MMA commits issued,
// [3] epilogue warp 2 past tfull-wait, [4] epilogue warp 2 arrived tempty
__device__ unsigned long long g_tile_ts[6][32];
// Compiled in only with -DB2_TILE_TS: the lane-0 branches inside the MMA issue
// loop cost ~7% on single-K-block GEMMs (they break the converged issuer).
B2_DEV void tile_stamp(const TcArgs& a, int which, int tile) {
#ifndef B2_TILE_TS
  return;
#endif
  if (TS_DBG(a) == 2 && blockIdx.x == 0 && tile < 32) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    g_tile_ts[which][tile] = g;
  }
}

B2_DEV void split_range(int s, int nsplit, int KT, int& kb0, int& kb1) {
  kb0 = (int)((long)s * KT / nsplit);
  kb1 = (int)((long)(s + 1) * KT / nsplit);
}

// M tile of linear tile index t.  Consecutive layers alternate the M
// direction (a.reverse): the next kernel then starts on the rows its producer
// wrote last, which are still in L2.
B2_DEV int mtile_of(const TcArgs& a, int t) {
  const int mt = t / a.tiles_n;
  return a.reverse ? a.tiles_m - 1 - mt : mt;
}

// Tiles t = t0, t0 + tstep, ... < ntiles; tile t covers rows
// (t / tiles_n) * mstride + mofs.  `tempty_remote` != 0: signal accumulator
// release on the CTA-pair leader's barrier (cluster address) instead of ours.
template <int BN, int ACT>
B2_DEV void epi_tma(const TcArgs& a, const CUtensorMap& tmO, uint8_t* sEpi, uint64_t* tfull,
                    uint64_t* tempty, uint32_t tmem_base, int ntiles, int lg, int ew, int eh,
                    int lane, int t0, int tstep, int mstride, int mofs, uint32_t tempty_remote) {
  const bool has_res = a.res != nullptr;
  int it = 0;
  // 32-column chunks split between the two warps of each TMEM lane
  // quadrant (chunk parity = warp half).  Per chunk: tcgen05.ld.x32, +bias,
  // +residual (prefetched one chunk ahead), act, bf16 pack into a
  // 64B-swizzled 32x32 staging tile, per-warp TMA store.
  uint8_t* obuf = sEpi + ew * 4096;
  uint32_t oi = 0;
  const uint32_t swz = (lane >> 1) & 3;
  for (int t = t0; t < ntiles; t += tstep, ++it) {
    const int as = it & 1;
    const uint32_t aph = (it >> 1) & 1;
    const int m0 = mtile_of(a, t) * mstride + mofs;
    const int n0 = (t % a.tiles_n) * BN;
    const int row0 = m0 + lg * 32;
    const int row = row0 + lane;
    const bool rvalid = row < a.M;
    const bf16* rrow = has_res ? a.res + (size_t)(rvalid ? row : 0) * a.ldres + n0 : nullptr;
    uint4 rnext[4];
    if (has_res) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        rnext[q] = (rvalid && n0 + eh * 32 + q * 8 < a.N)
                       ? __ldg(reinterpret_cast<const uint4*>(rrow + eh * 32) + q)
                       : make_uint4(0, 0, 0, 0);
    }
    // bias of the first chunk, fetched before the accumulator wait (a global
    // load per chunk on the critical path cost ~3 us per exposed tile)
    float4 bnext[8];
    {
      const float4* bp = reinterpret_cast<const float4*>(a.bias + n0 + eh * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) bnext[q] = a.bias ? __ldg(bp + q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    mbar_wait(&tfull[as], aph);
    tc_fence_after();
#ifdef B2_TILE_TS
    if (ew == 0 && lane == 0) tile_stamp(a, 3, it);
#endif
    const uint32_t taddr = tmem_base + (uint32_t(lg * 32) << 16) + as * BN;
#pragma unroll 1
    for (int c = eh * 32; c < BN && n0 + c < a.N; c += 64) {   // ragged N: skip empty chunks
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + c, r);
      uint4 rcur[4];
      if (has_res) {
#pragma unroll
        for (int q = 0; q < 4; ++q) rcur[q] = rnext[q];
        if (c + 64 < BN) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            rnext[q] = (rvalid && n0 + c + 64 + q * 8 < a.N)
                           ? __ldg(reinterpret_cast<const uint4*>(rrow + c + 64) + q)
                           : make_uint4(0, 0, 0, 0);
        }
      }
      float bv[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        bv[4 * q] = bnext[q].x;
        bv[4 * q + 1] = bnext[q].y;
        bv[4 * q + 2] = bnext[q].z;
        bv[4 * q + 3] = bnext[q].w;
      }
      if (c + 64 < BN && a.bias) {
        const float4* bp = reinterpret_cast<const float4*>(a.bias + n0 + c + 64);
#pragma unroll
        for (int q = 0; q < 8; ++q) bnext[q] = __ldg(bp + q);
      }
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int j = 0; j < 16; ++j)   // + bias on packed pairs (add.rn.f32x2: per-lane identical)
        f2unpack(f2add(f2pack(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])),
                       f2pack(bv[2 * j], bv[2 * j + 1])),
                 v[2 * j], v[2 * j + 1]);
      if (has_res) {
#pragma unroll
        for (int q = 0; q < 4; ++q) add_bf16x8(v + 8 * q, rcur[q]);
      }
      // GELU on packed pairs (f32x2 FMAs); other activations per element below
      constexpr int PACT = ACT == ACT_GELU ? ACT_NONE : ACT;
      if constexpr (ACT == ACT_GELU) {
#pragma unroll
        for (int j = 0; j < 16; ++j) gelu_erf2(v[2 * j], v[2 * j + 1]);
      }
      if (lane == 0 && EPI_DBG(a) != 4 && EPI_DBG(a) != 5) bulk_wait_read<1>();
      __syncwarp();
      uint8_t* sbuf = obuf + (oi & 1) * 2048;
      uint8_t* orow = sbuf + lane * 64;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (EPI_DBG(a) == 6) {
          if (v[q * 8] == 1234.5f) orow[q] = 1;
          continue;
        }
        uint4 u;
        u.x = act_pack2<PACT>(v[q * 8 + 0], v[q * 8 + 1]);
        u.y = act_pack2<PACT>(v[q * 8 + 2], v[q * 8 + 3]);
        u.z = act_pack2<PACT>(v[q * 8 + 4], v[q * 8 + 5]);
        u.w = act_pack2<PACT>(v[q * 8 + 6], v[q * 8 + 7]);
        *reinterpret_cast<uint4*>(orow + ((q ^ swz) << 4)) = u;
      }
      if (EPI_DBG(a) != 3) fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && EPI_DBG(a) != 5) {
        if (a.out3d)
          tma_store_3d(&tmO, sbuf, n0 + c, lg * 32, m0 / TC_BM);
        else
          tma_store_2d(&tmO, sbuf, n0 + c, row0);
        bulk_commit();
      }
      ++oi;
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (tempty_remote) mbar_arrive_cluster(tempty_remote + as * 8);
      else mbar_arrive(&tempty[as]);
#ifdef B2_TILE_TS
      if (ew == 0) tile_stamp(a, 4, it);
#endif
    }
  }
  if (lane == 0) bulk_wait<0>();
}

template <int BN, bool GATHER>
__global__ void __launch_bounds__(TcCfg<BN, GATHER>::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO,
                   const __grid_constant__ CUtensorMap tmR,
                   const __grid_constant__ CUtensorMap tmI, const TcArgs a) {
  using Cfg = TcCfg<BN, GATHER>;
  const int STAGES = a.stages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sEpi = sB + STAGES * Cfg::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + TC_EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_index_uniform();
  const int lane = threadIdx.x & 31;
  const int ntiles = a.tiles_m * a.tiles_n;
  // split-K (small batches): unit u = split (u / ntiles) of tile (u % ntiles);
  // each split stores its fp32 partial into its own workspace slice and
  // splitk_finalize sums the slices in order (deterministic) and applies
  // bias, residual, activation, bf16
  const int nunits = ntiles * a.nsplit;
  const int KT = a.kblocks + a.res_kblocks;

  __shared__ unsigned long long ts[8];    // B2_GEMM_TS phase timestamps (globaltimer, ns)
  auto stamp = [&](int i) {
    if (TS_DBG(a)) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      ts[i] = g;
    }
  };
  if (threadIdx.x == 0) {
    stamp(0);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], GATHER ? 1 + 128 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], TC_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    if (!GATHER) tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (a.res_kblocks) {
      tma_prefetch_desc(&tmR);
      tma_prefetch_desc(&tmI);
    }
    if (a.tma_epi) tma_prefetch_desc(&tmO);
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = uniform_u32(*tmem_slot);
  pdl_wait();                 // previous kernel's outputs (our A / residual) are complete
  pdl_launch_dependents();
  if (threadIdx.x == 0) stamp(1);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Whole warp converged, one elected lane issues (see the CTA-pair kernel:
    // warp-uniform operands, no per-TMA waterfall, no divisions per K block).
    const int Cin = a.C;
    const int Stap = a.S;
    const int kblocks = a.kblocks;
    const int im2col = a.a_im2col;
    const int fold = a.fold_kind;
    const uint32_t full_lo = uniform_u32(smem_u32(&full[0]));
    const uint32_t empty_lo = uniform_u32(smem_u32(&empty[0]));
    const uint32_t sA_lo = uniform_u32(smem_u32(sA)), sB_lo = uniform_u32(smem_u32(sB));
    const uint32_t a_bytes = GATHER ? 0u : (im2col == 0 && a.a_narrow)
                                               ? uint32_t(TC_BM * a.a_narrow * 2)
                                               : uint32_t(Cfg::A_BYTES);
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int t = u % ntiles;
      int kb0, kb1;
      split_range(u / ntiles, a.nsplit, KT, kb0, kb1);
      const int m0 = mtile_of(a, t) * TC_BM;
      const int n0 = (t % a.tiles_n) * BN;
      int iw0 = 0, ih0 = 0, img = 0;
      if (!GATHER && (im2col || fold == 2)) {
        img = m0 / a.OHW;
        const int rem = m0 - img * a.OHW;
        const int oh = rem / a.OW;
        ih0 = oh * a.stride;
        iw0 = (rem - oh * a.OW) * a.stride;
      }
      // im2col (mode 1) counters at K block kb0: channel offset and filter tap
      int c0 = 0, s2 = 0, r = 0;
      if (!GATHER && im2col == 1 && kb0 > 0 && kb0 < kblocks) {
        const int cpb = Cin >> 6;
        const int tap = kb0 / cpb;
        c0 = (kb0 - tap * cpb) << 6;
        r = tap / Stap;
        s2 = tap - r * Stap;
      }
      for (int kb = kb0; kb < kb1; ++kb) {
#ifdef B2_TILE_TS
        if (kb == kb0 && TS_DBG(a) == 2 && lane == 0)
          tile_stamp(a, 5, (u - (int)blockIdx.x) / (int)gridDim.x);
#endif
        mbar_wait_u32(empty_lo + stage * 8, phase ^ 1);
#ifdef B2_TILE_TS
        if (kb == kb0 && TS_DBG(a) == 2 && lane == 0)
          tile_stamp(a, 0, (u - (int)blockIdx.x) / (int)gridDim.x);
#endif
        const uint32_t fb = full_lo + stage * 8;
        const uint32_t dA = sA_lo + stage * Cfg::A_BYTES;
        const uint32_t dB = sB_lo + stage * Cfg::B_BYTES;
        if (elect_one()) {
          if (kb >= kblocks) {
            const int j = kb - kblocks;
            mbar_arrive_expect_tx_u32(fb, Cfg::A_BYTES + Cfg::B_BYTES);
            if (fold == 0) {
              // residual fold: A = res[m0:, n0 + j*64:], B = identity rows [0, BN)
              tma_load_2d_u32(dA, &tmR, fb, n0 + j * TC_BK, m0);
              tma_load_2d_u32(dB, &tmI, fb, j * TC_BK, 0);
            } else {
              // folded projection shortcut: A = its input x, B = its weights
              if (fold == 1)
                tma_load_2d_u32(dA, &tmR, fb, j * TC_BK, m0);
              else
                tma_load_im2col_4d_u32(dA, &tmR, fb, j * TC_BK, iw0, ih0, img, 0, 0);
              tma_load_2d_u32(dB, &tmI, fb, j * TC_BK, n0);
            }
          } else {
            if (GATHER) {
              mbar_arrive_expect_tx_u32(fb, Cfg::B_BYTES);
            } else if (im2col == 3) {
              // s2d stem: tile = output row (img, oh); K block kb = filter row-pair
              mbar_arrive_expect_tx_u32(fb, Cfg::A_BYTES + Cfg::B_BYTES);
              const int rt = m0 / TC_BM;
              const int im = rt / a.OH;
              tma_load_4d_u32(dA, &tmA, fb, 0, 0, rt - im * a.OH + kb, im);
            } else if (im2col == 2) {
              // 8 taps x (128 pixels x 8 channels); taps past R*S load tap 0
              // (finite data) against zero weights
              mbar_arrive_expect_tx_u32(fb, Cfg::A_BYTES + Cfg::B_BYTES);
              const int ntaps = a.R * a.S;
#pragma unroll 1
              for (int j = 0; j < 8; ++j) {
                int tap = kb * 8 + j;
                if (tap >= ntaps) tap = 0;
                const int rr = tap / a.S;
                const int ss = tap - rr * a.S;
                tma_load_im2col_4d_u32(dA + j * 2048, &tmA, fb, 0, iw0 - a.pad, ih0 - a.pad, img,
                                       (uint16_t)ss, (uint16_t)rr);
              }
            } else if (im2col) {
              mbar_arrive_expect_tx_u32(fb, Cfg::A_BYTES + Cfg::B_BYTES);
              tma_load_im2col_4d_u32(dA, &tmA, fb, c0, iw0 - a.pad, ih0 - a.pad, img,
                                     (uint16_t)s2, (uint16_t)r);
            } else {
              // narrow K: the A box is a_narrow elements wide (no out-of-bounds fill)
              mbar_arrive_expect_tx_u32(fb, a_bytes + Cfg::B_BYTES);
              tma_load_2d_u32(dA, &tmA, fb, kb * TC_BK, m0);
            }
            tma_load_2d_u32(dB, &tmB, fb, kb * TC_BK, n0);
          }
        }
        __syncwarp();
        if ((c0 += TC_BK) >= Cin) {
          c0 = 0;
          if (++s2 == Stap) {
            s2 = 0;
            ++r;
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // (whole warp, converged; one elected lane issues — see common.cuh)
    {
      constexpr uint32_t idesc = make_idesc(TC_BM, BN, 1u);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
        int kb0, kb1;
        split_range(u / ntiles, a.nsplit, KT, kb0, kb1);
        const int as = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem_base + as * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (it == 0 && kb == 0 && lane == 0) stamp(2);
#ifdef B2_TILE_TS
          if (kb == kb0 && lane == 0) tile_stamp(a, 1, it);
#endif
          const bool tap8 = a.a_im2col == 2 && kb < a.kblocks;
          const bool narrow = a.a_narrow && kb < a.kblocks;
          const uint32_t a_addr = smem_u32(sA + stage * Cfg::A_BYTES);
          const uint64_t ad = tap8 ? smem_desc_kmajor_noswizzle(a_addr, 2048, 128)
                              : narrow ? (a.a_narrow == 32 ? smem_desc_sw64_k(a_addr)
                                                           : smem_desc_sw32_k(a_addr))
                                       : smem_desc_sw128(a_addr);
          const uint32_t astep = tap8 ? 256u : 2u;   // K += 16: 2 taps (4 KB) or 32 B
          const int ksteps = narrow ? a.a_narrow / 16 : TC_BK / 16;
          const uint64_t bd = smem_desc_sw128(smem_u32(sB + stage * Cfg::B_BYTES));
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            if (k < ksteps && elect_one())
              umma_bf16(dt, ad + astep * k, bd + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          if (elect_one()) umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit(&tfull[as]);
#ifdef B2_TILE_TS
        if (lane == 0) tile_stamp(a, 2, it);
#endif
      }
      if (lane == 0) stamp(3);
    }
  } else if (warp < 2 + TC_EPI_WARPS) {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3;          // TMEM lane quadrant this warp may access
    const int ew = warp - 2;
    const int eh = ew >> 2;           // which half of each quadrant's columns
    const bool has_res = a.res != nullptr;
    int it = 0;
    if (EPI_DBG(a) == 1) {
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int as = it & 1;
        mbar_wait(&tfull[as], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t(lg * 32) << 16) + as * BN;
        uint32_t acc = 0;
        for (int c = eh * 32; c + 32 <= BN; c += 64) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c, r);
          tmem_wait_ld();
          acc ^= r[0] ^ r[31];
        }
        if (acc == 0x7f7f7f7fu) a.out[0] = __float2bfloat16_rn(0.f);   // keep the loads alive
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[as]);
      }
    } else if (a.nsplit > 1) {
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
        const int t = u % ntiles;
        const int as = it & 1;
        mbar_wait(&tfull[as], (it >> 1) & 1);
        tc_fence_after();
        const int row = mtile_of(a, t) * TC_BM + lg * 32 + lane;
        const int n0 = (t % a.tiles_n) * BN;
        const uint32_t taddr = tmem_base + (uint32_t(lg * 32) << 16) + as * BN;
#pragma unroll 1
        for (int c = eh * 32; c < BN && n0 + c < a.N; c += 64) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(taddr + c, r);
          tmem_wait_ld();
          if (row < a.M) {   // this split's slice: deterministic order
            float4* dst = reinterpret_cast<float4*>(
                a.ws + ((size_t)(u / ntiles) * a.M + row) * a.N + n0 + c);
#pragma unroll
            for (int q = 0; q < 8; ++q)   // ragged last N tile: columns < N only (N % 8 == 0)
              if (n0 + c + 4 * q < a.N)
                dst[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                     __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[as]);
      }
    } else if (BN >= 32 && a.tma_epi) {
      switch (a.act) {
        case ACT_RELU: epi_tma<BN, ACT_RELU>(a, tmO, sEpi, tfull, tempty, tmem_base, ntiles, lg, ew, eh, lane, blockIdx.x, gridDim.x, TC_BM, 0, 0u); break;
        case ACT_RELU6: epi_tma<BN, ACT_RELU6>(a, tmO, sEpi, tfull, tempty, tmem_base, ntiles, lg, ew, eh, lane, blockIdx.x, gridDim.x, TC_BM, 0, 0u); break;
        case ACT_GELU: epi_tma<BN, ACT_GELU>(a, tmO, sEpi, tfull, tempty, tmem_base, ntiles, lg, ew, eh, lane, blockIdx.x, gridDim.x, TC_BM, 0, 0u); break;
        case ACT_TANH: epi_tma<BN, ACT_TANH>(a, tmO, sEpi, tfull, tempty, tmem_base, ntiles, lg, ew, eh, lane, blockIdx.x, gridDim.x, TC_BM, 0, 0u); break;
        default: epi_tma<BN, ACT_NONE>(a, tmO, sEpi, tfull, tempty, tmem_base, ntiles, lg, ew, eh, lane, blockIdx.x, gridDim.x, TC_BM, 0, 0u); break;
      }
    } else {
      // direct path (narrow tiles / N not a multiple of 8): 16-byte stores
      const bool vec_ok = (a.ldo % 8 == 0) && (!has_res || a.ldres % 8 == 0);
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int as = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        const int m0 = mtile_of(a, t) * TC_BM;
        const int n0 = (t % a.tiles_n) * BN;
        mbar_wait(&tfull[as], aph);
        tc_fence_after();
        const int row = m0 + lg * 32 + lane;
        const uint32_t taddr = tmem_base + (uint32_t(lg * 32) << 16) + as * BN;
        constexpr int CH = BN >= 32 ? 32 : BN;
#pragma unroll 1
        for (int c = eh * CH; c < BN; c += 2 * CH) {
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
              for (int j = 0; j < CH; ++j)
                if (a.bias) v[j] += __ldg(a.bias + col0 + j);
              if (has_res) {
                const uint4* rp =
                    reinterpret_cast<const uint4*>(a.res + (size_t)row * a.ldres + col0);
#pragma unroll
                for (int q = 0; q < CH / 8; ++q) add_bf16x8(v + 8 * q, __ldg(rp + q));
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
                if (has_res) x += __bfloat162float(a.res[(size_t)row * a.ldres + col]);
                a.out[(size_t)row * a.ldo + col] = __float2bfloat16_rn(act_apply(x, a.act));
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[as]);
      }
    }
  } else if (GATHER) {
    // ------------------------------------------------------------ im2col gather
    const int g = threadIdx.x - (2 + TC_EPI_WARPS) * 32;   // A-tile row owned by this thread
    const uint32_t sw = g & 7;
    int stage = 0;
    uint32_t phase = 0;
    const size_t img_elems = (size_t)a.H * a.W * a.C;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int m = mtile_of(a, t) * TC_BM + g;
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
        if (a.gmode == 2) {
          // S*C <= 64: K block kb is filter row r = kb; its S taps are one
          // contiguous run of S*C channels starting at input column iw0
          const int ih = ih0 + kb;
          const bool rok = vrow && (unsigned)ih < (unsigned)a.H;
          const bf16* rowp = xb + ((long)ih * a.W + iw0) * a.C;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int e = j * 8;
            const int s = e >> a.c_log2;
            const bool ok = rok && e < a.SC && (unsigned)(iw0 + s) < (unsigned)a.W;
            cp_async_16(dst + ((j ^ sw) << 4), ok ? rowp + e : a.x, ok ? 16u : 0u);
          }
        } else if (a.gmode == 1) {
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
        cp_async_mbar_arrive(&full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      for (int j = 0; j < a.res_kblocks; ++j) {   // residual-fold stages: TMA fills A
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive(&full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    cp_async_wait<0>();
  }

  if (warp == 2 && lane == 0) stamp(4);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && TS_DBG(a)) {
    stamp(5);
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("b2ts %d %u %llu %llu %llu %llu %llu %llu stages %d kblocks %d tiles %d\n", blockIdx.x,
           smid, ts[0], ts[1], ts[2], ts[3], ts[4], ts[5], STAGES, a.kblocks, ntiles);
#ifdef B2_TILE_TS
    if (TS_DBG(a) == 2 && blockIdx.x == 0)
#else
    if (false)
#endif
      for (int t = 0; t < 32; ++t)
        printf("b2tile %d %llu %llu %llu %llu %llu %llu\n", t, g_tile_ts[0][t], g_tile_ts[1][t],
               g_tile_ts[2][t], g_tile_ts[3][t], g_tile_ts[4][t], g_tile_ts[5][t]);
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ============================================================================
// CTA-pair GEMM (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x BN tile with M = 256 UMMAs issued by the leader.  Each CTA loads its
// own 128 A rows and HALF of the BN weight rows; the MMA reads the other half
// from the peer's shared memory.  Per SM this halves the weight traffic and
// the weight smem per stage (A 16 KB + B BN/2 x 128 B), so the ring is ~1.5x
// deeper for the same MMA work — the late-ResNet / BERT GEMMs are bound by
// operand delivery, not by the tensor pipe (ncu: MMA thread waiting on TMA
// ~45% with 128 x 256 single-CTA tiles).
//
// Barriers: full[s] lives in the leader (both CTAs' TMA loads complete_tx on
// it, the leader alone expects 2 x stage bytes); empty[s] and tfull[] exist in
// both CTAs and receive the leader's multicast commits; the leader's
// tempty[] collects the epilogue warps of both CTAs (16 arrivals).
template <int BN>
struct Tc2Cfg {
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = (BN / 2) * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (TC_SMEM_MAX - TC_EPI_BYTES - 1024 - TC_BAR_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 10 ? 10 : STAGES_RAW;
  static constexpr int THREADS = (2 + TC_EPI_WARPS) * 32;
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + TC_EPI_BYTES + 1024 + TC_BAR_BYTES;
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Tc2Cfg<BN>::THREADS, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap tmA,
                    const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmO,
                    const __grid_constant__ CUtensorMap tmR,
                    const __grid_constant__ CUtensorMap tmI, const TcArgs a) {
  using Cfg = Tc2Cfg<BN>;
  constexpr int ST = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST * Cfg::A_BYTES;
  uint8_t* sEpi = sB + ST * Cfg::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + TC_EPI_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_index_uniform();
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int ntiles = a.tiles_m * a.tiles_n;
  const int KT = a.kblocks + a.res_kblocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * TC_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (a.res_kblocks) {
      tma_prefetch_desc(&tmR);
      tma_prefetch_desc(&tmI);
    }
    tma_prefetch_desc(&tmO);
  }
  cluster_sync();                       // barrier inits visible to the peer
  if (warp == 1) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = uniform_u32(*tmem_slot);
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    // The whole warp runs the loop converged and one elected lane issues:
    // every value below derives from kernel parameters, blockIdx and loop
    // counters (warp-uniform), so the TMA operands live in uniform registers.
    // (A single-lane producer paid an ELECT/R2UR waterfall per TMA, two integer
    // divisions and constant-bank reloads per K block, ~100 SASS per 512-clock
    // K block: ncu showed it never waiting for a free ring slot while the MMA
    // thread spun on full barriers — the producer paced the kernel.)  Per K
    // block now: the empty wait, address adds, the loads, and im2col taps
    // advanced as counters.
    const int Cin = a.C;
    const int Stap = a.S;
    const int kblocks = a.kblocks;
    const bool im2col = a.a_im2col != 0;
    const int fold = a.fold_kind;
    const int urank = (int)uniform_u32(rank);
    const uint32_t full_cl = uniform_u32(mapa_shared(&full[0], 0));   // the leader's full[0]
    const uint32_t full_lo = uniform_u32(smem_u32(&full[0]));
    const uint32_t empty_lo = uniform_u32(smem_u32(&empty[0]));
    const uint32_t sA_lo = uniform_u32(smem_u32(sA)), sB_lo = uniform_u32(smem_u32(sB));
    int stage = 0;
    uint32_t phase = 0;
    for (int t = cid; t < ntiles; t += ncl) {
      const int m0 = mtile_of(a, t) * (2 * TC_BM) + urank * TC_BM;
      const int n0 = (t % a.tiles_n) * BN;
      const int nb = n0 + urank * (BN / 2);          // this CTA's half of the weights
      int iw0 = 0, ih0 = 0, img = 0;
      if (im2col || fold == 2) {
        img = m0 / a.OHW;
        const int rem = m0 - img * a.OHW;
        const int oh = rem / a.OW;
        ih0 = oh * a.stride;
        iw0 = (rem - oh * a.OW) * a.stride;
      }
      int c0 = 0, s2 = 0, r = 0;                      // im2col: channel block, filter tap
      for (int kb = 0; kb < KT; ++kb) {
        mbar_wait_u32(empty_lo + stage * 8, phase ^ 1);
        const uint32_t fl = full_cl + stage * 8;
        const uint32_t dA = sA_lo + stage * Cfg::A_BYTES;
        const uint32_t dB = sB_lo + stage * Cfg::B_BYTES;
        if (elect_one()) {
          if (urank == 0) mbar_arrive_expect_tx_u32(full_lo + stage * 8, 2 * Cfg::STAGE_BYTES);
          if (kb >= kblocks) {
            const int j = kb - kblocks;
            if (fold == 0) {   // residual x identity (this CTA's half of the rows)
              tma_load_2d_pair_u32(dA, &tmR, fl, n0 + j * TC_BK, m0);
              tma_load_2d_pair_u32(dB, &tmI, fl, j * TC_BK, urank * (BN / 2));
            } else {           // folded projection shortcut: x (or strided x) x Wd
              if (fold == 1)
                tma_load_2d_pair_u32(dA, &tmR, fl, j * TC_BK, m0);
              else
                tma_load_im2col_4d_pair_u32(dA, &tmR, fl, j * TC_BK, iw0, ih0, img, 0, 0);
              tma_load_2d_pair_u32(dB, &tmI, fl, j * TC_BK, nb);
            }
          } else {
            if (im2col)
              tma_load_im2col_4d_pair_u32(dA, &tmA, fl, c0, iw0 - a.pad, ih0 - a.pad, img,
                                          (uint16_t)s2, (uint16_t)r);
            else
              tma_load_2d_pair_u32(dA, &tmA, fl, kb * TC_BK, m0);
            tma_load_2d_pair_u32(dB, &tmB, fl, kb * TC_BK, nb);
          }
        }
        __syncwarp();
        if ((c0 += TC_BK) >= Cin) {
          c0 = 0;
          if (++s2 == Stap) {
            s2 = 0;
            ++r;
          }
        }
        if (++stage == ST) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader, whole warp)
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc(2 * TC_BM, BN, 1u);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cid; t < ntiles; t += ncl, ++it) {
        const int as = it & 1;
        mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem_base + as * BN;
        for (int kb = 0; kb < KT; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(smem_u32(sA + stage * Cfg::A_BYTES));
          const uint64_t bd = smem_desc_sw128(smem_u32(sB + stage * Cfg::B_BYTES));
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            if (elect_one()) umma_bf16_pair(dt, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          if (elect_one()) umma_commit_pair(&empty[stage]);
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_pair(&tfull[as]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int lg = warp & 3;
    const int ew = warp - 2;
    const int eh = ew >> 2;
    const uint32_t trem = rank == 0 ? 0u : mapa_shared(&tempty[0], 0);
    switch (a.act) {
#define B2_EPI2(ACTV)                                                                            \
  epi_tma<BN, ACTV>(a, tmO, sEpi, tfull, tempty, tmem_base, ntiles, lg, ew, eh, lane, cid, ncl, \
                    2 * TC_BM, (int)rank * TC_BM, trem)
      case ACT_RELU: B2_EPI2(ACT_RELU); break;
      case ACT_RELU6: B2_EPI2(ACT_RELU6); break;
      case ACT_GELU: B2_EPI2(ACT_GELU); break;
      case ACT_TANH: B2_EPI2(ACT_TANH); break;
      default: B2_EPI2(ACT_NONE); break;
#undef B2_EPI2
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();                       // the peer is done with our barriers and TMEM
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side

template <int BN, bool G>
static cudaError_t launch_bn(TcArgs a, const CUtensorMap& ta, const CUtensorMap& tb,
                             const CUtensorMap& to, const CUtensorMap& tr, const CUtensorMap& ti,
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
  if (a.stages <= 0 || a.stages > Cfg::MAX_STAGES) a.stages = Cfg::MAX_STAGES;
  const int units = a.tiles_m * a.tiles_n * a.nsplit;
  const int grid = units < num_sms ? units : num_sms;
  return launch_pdl(kern, dim3(grid), dim3(Cfg::THREADS), Cfg::SMEM, st, ta, tb, to, tr, ti, a);
}

template <int BN>
static cudaError_t launch_pair(TcArgs a, const CUtensorMap& ta, const CUtensorMap& tb,
                               const CUtensorMap& to, const CUtensorMap& tr, const CUtensorMap& ti,
                               int num_sms, cudaStream_t st) {
  using Cfg = Tc2Cfg<BN>;
  auto kern = tc_gemm2_kernel<BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int tiles = a.tiles_m * a.tiles_n;
  const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
  return launch_pdl(kern, dim3(2 * pairs), dim3(Cfg::THREADS), Cfg::SMEM, st, ta, tb, to, tr, ti,
                    a);
}

// CTA-pair launch: a.tiles_m counts 256-row pair tiles; tb / ti boxes are BN/2 rows.
cudaError_t tc_gemm2_launch(const TcArgs& a, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                            const CUtensorMap& to, const CUtensorMap& tr, const CUtensorMap& ti,
                            int num_sms, cudaStream_t st) {
  if (bn == 256) return launch_pair<256>(a, ta, tb, to, tr, ti, num_sms, st);
  if (bn == 128) return launch_pair<128>(a, ta, tb, to, tr, ti, num_sms, st);
  return cudaErrorInvalidValue;
}

// BN for the CTA-pair kernel: fewest pair-tile waves, MMA time per tile ~ BN.
int tc2_pick_bn(long M, int N, int num_sms) {
  const long tm = (M + 2 * TC_BM - 1) / (2 * TC_BM);
  const int pairs = num_sms / 2;
  long best_cost = -1;
  int best = 0;
  for (int bn : {256, 128}) {
    if (bn / 2 >= N) continue;
    const long tiles = tm * ((N + bn - 1) / bn);
    const long cost = (tiles + pairs - 1) / pairs * bn;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

// Split-K factor for small batches: when the tiles cannot fill half the SMs
// and the K loop is long, spread each tile's K over up to 16 CTAs (>= 4 K
// blocks each).  Large batches keep nsplit = 1.
int tc_pick_split(long tiles, int kt, int num_sms) {
  if (tiles * 2 > num_sms || kt < 8) return 1;
  int sp = (int)(num_sms / tiles);
  if (sp > kt / 4) sp = kt / 4;
  if (sp > 16) sp = 16;
  return sp < 2 ? 1 : sp;
}

// Tile shape + kernel (single CTA vs CTA pair) from a per-SM clock model.
// Per 64-wide K block a tile costs max(MMA, operand bytes / TMA rate): the
// chip's TMA/L2 fill rate (~12 TB/s measured, ~42 B/clk per SM) is below what
// a 128 x 256 tile's MMAs consume (48 KB per 512 MMA clocks), so the CTA pair
// -- each CTA loads its own A rows but only half of B -- runs long-K shapes
// ~1.5x faster. The epilogue (~10.5 B/clk of output per SM) overlaps the next
// tile's mainloop, so short-K tiles cost max(mainloop, epilogue).
// Measured at M = 16384, K = 768: N = 2304 62.8 -> 50.2 us, N = 3072 (was
// BN = 128 single) 127 -> see DESIGN.md; K = 256 N = 1024 stays single.
static double tc_tile_clk(int bn, bool pair, int kblocks, int nvalid) {
  const double mma = 4.0 * (bn > 128 ? 128 : 64);
  const double bytes = 16384.0 + (pair ? bn / 2 : bn) * 128.0;
  const double mainloop = kblocks * (mma > bytes / 42.0 ? mma : bytes / 42.0);
  const double epi = 128.0 * (nvalid < bn ? nvalid : bn) * 2.0 / 10.5;
  // + ~600 clk per tile of barrier round trips / TMEM hand-off / pipeline
  // refill that no overlap hides (keeps narrow tiles from winning ties)
  return (mainloop > epi ? mainloop : epi) + 600.0;
}

int tc_pick_config(long M, int N, int kblocks, bool res_fold, int num_sms, bool pair_allowed,
                   bool* pair_out) {
  const int cands[5] = {256, 128, 64, 32, 16};
  double best_cost = -1;
  int best = 16;
  bool best_pair = false;
  for (int pass = 0; pass < 2; ++pass) {
    const bool pair = pass == 1;
    if (pair && !pair_allowed) break;
    for (int bn : cands) {
      if (pair && bn < 128) continue;
      if (bn > 16 && bn / 2 >= N && !(bn == 32 && N % 8 == 0 && N >= 8)) continue;
      if (bn == 16 && N % 8 == 0) continue;   // BN = 32 gets the TMA-store epilogue
      const long tm = pair ? (M + 2 * TC_BM - 1) / (2 * TC_BM) : (M + TC_BM - 1) / TC_BM;
      const long tn = (N + bn - 1) / bn;
      const long slots = pair ? num_sms / 2 : num_sms;
      const long waves = (tm * tn + slots - 1) / slots;
      const int kb = kblocks + (res_fold ? (bn >= 64 ? bn / 64 : 1) : 0);
      const double cost = waves * tc_tile_clk(bn, pair, kb, (int)(N / tn));   // mean valid cols
      if (best_cost < 0 || cost < best_cost * 0.999) {
        best_cost = cost;
        best = bn;
        best_pair = pair;
      }
    }
  }
  *pair_out = best_pair;
  return best;
}

int tc_pick_bn(long M, int N, int num_sms) {
  const int cands[5] = {256, 128, 64, 32, 16};
  long best_cost = -1;
  int best = 16;
  const long tm = (M + TC_BM - 1) / TC_BM;
  for (int bn : cands) {
    // far wider than N: wasted columns -- except BN = 32 for N = 16..31 with
    // N % 8 == 0: same MMA cost as BN = 16 but the TMA-store epilogue (the
    // per-thread row stores of the narrow path measured 248 vs ~70 us at
    // M = 3.2M, K = 32, N = 16)
    if (bn > 16 && bn / 2 >= N && !(bn == 32 && N % 8 == 0 && N >= 8)) continue;
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
                           const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& tr,
                           const CUtensorMap& ti, int num_sms, cudaStream_t st) {
#define B2_TC_CASE(BNV)                                                        \
  case BNV:                                                                    \
    return gather ? launch_bn<BNV, true>(a, ta, tb, to, tr, ti, num_sms, st)   \
                  : launch_bn<BNV, false>(a, ta, tb, to, tr, ti, num_sms, st);
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
