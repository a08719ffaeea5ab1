// Chained 1x1 convolutions on tcgen05 (sm_100a): a ResNet bottleneck's last
// conv and the NEXT block's first conv in one kernel,
//
//   O  = relu(T2 W3^T + b3 + R)          [M x N1]  (R: residual, or a folded
//                                                   projection shortcut x Wd^T)
//   T1 = relu(O  W1^T + b1)               [M x N2]  (N2 <= 256)
//
// O is still written (it is the next residual) but never read back: each
// 128-row tile of O is produced in 128-column chunks, converted to bf16 by
// the epilogue straight into shared memory in the 128B-swizzled K-major UMMA
// layout — which is also the TMA-store layout — so the same bytes are stored
// to HBM and consumed as the A operand of the second GEMM.  Saves one full
// read of every 256..1024-channel block output (411 MB at layer1, b=256) and
// one kernel per block.
//
// TMEM: two 128-column accumulators for O chunks (double buffered, so the
// first GEMM of chunk c+1 overlaps the epilogue of chunk c) + N2 columns for
// T1.  MMA order per tile: G1(0), G1(1), G2(0), G1(2), G2(1), ..., G2(C-1):
// the second GEMM trails by one chunk so the tensor pipe never waits for the
// epilogue.  Warp roles as in gemm_tc.cu: warp 0 TMA producer, warp 1 MMA
// issuer (converged, elected lane), warps 2..9 epilogue.
#include "common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int CH_BM = 128;
constexpr int CH_BN = 128;                   // O chunk width
constexpr int CH_BK = 64;
constexpr int CH_EPI_WARPS = 8;
constexpr int CH_THREADS = (2 + CH_EPI_WARPS) * 32;
constexpr int CH_SMEM_MAX = 232448;
constexpr int CH_A_BYTES = CH_BM * CH_BK * 2;        // 16 KB
constexpr int CH_B1_BYTES = CH_BN * CH_BK * 2;       // 16 KB
constexpr int CH_STAGE = CH_A_BYTES + CH_B1_BYTES;
constexpr int CH_A2_BYTES = CH_BM * CH_BN * 2;       // one O chunk: 2 K blocks of 16 KB

B2_DEV void chain_bar() { asm volatile("bar.sync 1, %0;" ::"n"(CH_EPI_WARPS * 32) : "memory"); }

B2_DEV uint32_t relu_pack2(float2 s) { return act_pack2<ACT_RELU>(s.x, s.y); }

B2_DEV int chain_mtile(const ChainArgs& a, int t) { return a.reverse ? a.tiles_m - 1 - t : t; }

__global__ void __launch_bounds__(CH_THREADS, 1)
    chain_gemm_kernel(const __grid_constant__ CUtensorMap tmA,    // T2 [M, K1]
                      const __grid_constant__ CUtensorMap tmB1,   // W3 [N1, K1], box 128 rows
                      const __grid_constant__ CUtensorMap tmR,    // residual / shortcut input
                      const __grid_constant__ CUtensorMap tmI,    // identity / shortcut weights
                      const __grid_constant__ CUtensorMap tmB2,   // W1 [N2, N1], box N2 rows
                      const __grid_constant__ CUtensorMap tmO,    // O  [M, N1], 64 x 128 SW128
                      const __grid_constant__ CUtensorMap tmT,    // T1 [M, N2], 64 x 128 SW128
                      const ChainArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int ST = a.stages, S2 = a.b2_stages;
  const int B2_BYTES = a.N2 * CH_BK * 2;
  uint8_t* sRing = smem;                                   // ST x (A 16 KB | B1 16 KB)
  uint8_t* sA2 = sRing + ST * CH_STAGE;                    // 2 x O chunk (32 KB each)
  uint8_t* sB2 = sA2 + 2 * CH_A2_BYTES;                    // S2 x (N2 x 64) weights
  // T1 staging of its own (N2 / 64 blocks of 16 KB): the T1 epilogue no longer
  // drains every outstanding O store before reusing the O buffers, and no
  // longer waits for its own store before the next tile's first O chunk
  uint8_t* sT = sB2 + S2 * B2_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sT + (a.N2 / 64) * CH_A_BYTES);
  uint64_t* empty = full + ST;
  uint64_t* b2full = empty + ST;
  uint64_t* b2empty = b2full + S2;
  uint64_t* c1full = b2empty + S2;       // [2] O chunk accumulator ready
  uint64_t* c1empty = c1full + 2;        // [2] O chunk accumulator drained (8 warps)
  uint64_t* a2full = c1empty + 2;        // [2] bf16 O chunk staged in smem (8 warps)
  uint64_t* a2empty = a2full + 2;        // [2] second GEMM done reading the chunk
  uint64_t* t2full = a2empty + 2;        // T1 accumulator ready
  uint64_t* t2empty = t2full + 1;        // T1 accumulator drained (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t2empty + 1);

  const int warp = warp_index_uniform();
  const int lane = threadIdx.x & 31;
  const int C = a.N1 / CH_BN;                      // O chunks per tile
  const int KT1 = a.kblocks + a.res_kblocks;       // first-GEMM K blocks per chunk
  const int KT2 = CH_BN / CH_BK;                   // second-GEMM K blocks per chunk (2)

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < S2; ++s) {
      mbar_init(&b2full[s], 1);
      mbar_init(&b2empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&c1full[i], 1);
      mbar_init(&c1empty[i], CH_EPI_WARPS);
      mbar_init(&a2full[i], CH_EPI_WARPS);
      mbar_init(&a2empty[i], 1);
    }
    mbar_init(t2full, 1);
    mbar_init(t2empty, CH_EPI_WARPS);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB1);
    tma_prefetch_desc(&tmR);
    tma_prefetch_desc(&tmI);
    tma_prefetch_desc(&tmB2);
    tma_prefetch_desc(&tmO);
    tma_prefetch_desc(&tmT);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = uniform_u32(*tmem_slot);
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t tacc2 = tmem_base + 2 * CH_BN;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // whole warp converged, one elected lane issues (warp-uniform operands, no
    // per-TMA ELECT/R2UR waterfall; see gemm_tc.cu's producers)
    {
      int st = 0, s2 = 0;
      uint32_t ph = 0, ph2 = 0;
      const int kblocks = a.kblocks, fold = a.fold_kind;
      const uint32_t full_lo = uniform_u32(smem_u32(&full[0]));
      const uint32_t empty_lo = uniform_u32(smem_u32(&empty[0]));
      const uint32_t b2full_lo = uniform_u32(smem_u32(&b2full[0]));
      const uint32_t b2empty_lo = uniform_u32(smem_u32(&b2empty[0]));
      const uint32_t ring_lo = uniform_u32(smem_u32(sRing));
      const uint32_t sB2_lo = uniform_u32(smem_u32(sB2));
      auto load_g1 = [&](int m0, int c, int fw, int fh, int fim) {
        const int n0 = c * CH_BN;
        for (int kb = 0; kb < KT1; ++kb) {
          mbar_wait_u32(empty_lo + st * 8, ph ^ 1);
          const uint32_t dA = ring_lo + st * CH_STAGE;
          const uint32_t dB = dA + CH_A_BYTES;
          const uint32_t fb = full_lo + st * 8;
          if (elect_one()) {
            mbar_arrive_expect_tx_u32(fb, CH_STAGE);
            if (kb < kblocks) {
              tma_load_2d_u32(dA, &tmA, fb, kb * CH_BK, m0);
              tma_load_2d_u32(dB, &tmB1, fb, kb * CH_BK, n0);
            } else {
              const int j = kb - kblocks;
              if (fold == 0) {                  // residual x identity
                tma_load_2d_u32(dA, &tmR, fb, n0 + j * CH_BK, m0);
                tma_load_2d_u32(dB, &tmI, fb, j * CH_BK, 0);
              } else {                          // projection shortcut x Wd
                if (fold == 1)
                  tma_load_2d_u32(dA, &tmR, fb, j * CH_BK, m0);
                else
                  tma_load_im2col_4d_u32(dA, &tmR, fb, j * CH_BK, fw, fh, fim, 0, 0);
                tma_load_2d_u32(dB, &tmI, fb, j * CH_BK, n0);
              }
            }
          }
          __syncwarp();
          if (++st == ST) {
            st = 0;
            ph ^= 1;
          }
        }
      };
      auto load_g2 = [&](int c) {
        for (int kb = 0; kb < KT2; ++kb) {
          mbar_wait_u32(b2empty_lo + s2 * 8, ph2 ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx_u32(b2full_lo + s2 * 8, (uint32_t)B2_BYTES);
            tma_load_2d_u32(sB2_lo + s2 * B2_BYTES, &tmB2, b2full_lo + s2 * 8,
                            c * CH_BN + kb * CH_BK, 0);
          }
          __syncwarp();
          if (++s2 == S2) {
            s2 = 0;
            ph2 ^= 1;
          }
        }
      };
      for (int t = blockIdx.x; t < a.tiles_m; t += gridDim.x) {
        const int m0 = chain_mtile(a, t) * CH_BM;
        int fw = 0, fh = 0, fim = 0;     // strided shortcut: its input pixel of row m0
        if (fold == 2) {
          fim = m0 / a.OHW;
          const int rem = m0 - fim * a.OHW;
          const int oh = rem / a.OW;
          fw = (rem - oh * a.OW) * a.stride;
          fh = oh * a.stride;
        }
        load_g1(m0, 0, fw, fh, fim);
        for (int c = 1; c < C; ++c) {
          load_g1(m0, c, fw, fh, fim);
          load_g2(c - 1);
        }
        load_g2(C - 1);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc1 = make_idesc(CH_BM, CH_BN, 1u);
    const uint32_t idesc2 = make_idesc(CH_BM, a.N2, 1u);
    int st = 0, s2 = 0;
    uint32_t ph = 0, ph2 = 0;
    int g = 0;         // global O-chunk counter (accumulator / staging buffer = g & 1)
    int tt = 0;        // tiles done by this CTA
    auto mma_g1 = [&](int gc) {
      const int buf = gc & 1;
      mbar_wait(&c1empty[buf], ((gc >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + buf * CH_BN;
      for (int kb = 0; kb < KT1; ++kb) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        const uint64_t ad = smem_desc_sw128(smem_u32(sRing + st * CH_STAGE));
        const uint64_t bd = smem_desc_sw128(smem_u32(sRing + st * CH_STAGE + CH_A_BYTES));
#pragma unroll
        for (int k = 0; k < CH_BK / 16; ++k)
          if (elect_one()) umma_bf16(d, ad + 2 * k, bd + 2 * k, idesc1, (kb | k) != 0 ? 1u : 0u);
        if (elect_one()) umma_commit(&empty[st]);
        if (++st == ST) {
          st = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) umma_commit(&c1full[buf]);
    };
    auto mma_g2 = [&](int gc, bool first) {
      const int buf = gc & 1;
      mbar_wait(&a2full[buf], (gc >> 1) & 1);
      tc_fence_after();
      for (int kb = 0; kb < KT2; ++kb) {
        mbar_wait(&b2full[s2], ph2);
        tc_fence_after();
        const uint64_t ad = smem_desc_sw128(smem_u32(sA2 + buf * CH_A2_BYTES + kb * CH_A_BYTES));
        const uint64_t bd = smem_desc_sw128(smem_u32(sB2 + s2 * B2_BYTES));
#pragma unroll
        for (int k = 0; k < CH_BK / 16; ++k)
          if (elect_one())
            umma_bf16(tacc2, ad + 2 * k, bd + 2 * k, idesc2, (first && kb == 0 && k == 0) ? 0u : 1u);
        if (elect_one()) umma_commit(&b2empty[s2]);
        if (++s2 == S2) {
          s2 = 0;
          ph2 ^= 1;
        }
      }
      if (elect_one()) umma_commit(&a2empty[buf]);
    };
    for (int t = blockIdx.x; t < a.tiles_m; t += gridDim.x, ++tt) {
      // the T1 accumulator is only needed by the second GEMM: wait for the
      // previous tile's T1 epilogue there, not before this tile's first GEMM
      auto wait_t2 = [&]() {
        mbar_wait(t2empty, (tt & 1) ^ 1);
        tc_fence_after();
      };
      mma_g1(g);
      for (int c = 1; c < C; ++c) {
        mma_g1(g + c);
        if (c == 1) wait_t2();
        mma_g2(g + c - 1, c == 1);
      }
      if (C == 1) wait_t2();
      mma_g2(g + C - 1, C == 1);
      if (elect_one()) umma_commit(t2full);
      g += C;
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                  // TMEM lane quadrant = tile rows q*32..
    const int eh = (warp - 2) >> 2;          // column half of each 64-column K block
    const int row = q * 32 + lane;           // tile row owned by this thread
    const bool issuer = warp == 2 && lane == 0;
    const uint32_t sw = row & 7;
    int g = 0, tt = 0;
    for (int t = blockIdx.x; t < a.tiles_m; t += gridDim.x, ++tt) {
      const int m0 = chain_mtile(a, t) * CH_BM;
      for (int c = 0; c < C; ++c, ++g) {
        const int buf = g & 1;
        mbar_wait(&c1full[buf], (g >> 1) & 1);
        tc_fence_after();
        // staging buffer free: second GEMM of chunk g-2 done, its O store read out
        mbar_wait(&a2empty[buf], ((g >> 1) & 1) ^ 1);
        if (issuer) bulk_wait_read<1>();
        chain_bar();
        uint8_t* dst = sA2 + buf * CH_A2_BYTES;
#pragma unroll 1
        for (int kb = 0; kb < 2; ++kb) {               // the chunk's two 64-column K blocks
          const int col = kb * 64 + eh * 32;           // this warp's 32 columns
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + buf * CH_BN + col, r);
          float bv[32];
          const float4* bp = reinterpret_cast<const float4*>(a.bias1 + c * CH_BN + col);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 b4 = __ldg(bp + j);
            bv[4 * j] = b4.x;
            bv[4 * j + 1] = b4.y;
            bv[4 * j + 2] = b4.z;
            bv[4 * j + 3] = b4.w;
          }
          tmem_wait_ld();
          uint8_t* rowp = dst + kb * CH_A_BYTES + row * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 w;
            w.x = relu_pack2(acc_add2(r[8 * j + 0], r[8 * j + 1], bv[8 * j + 0], bv[8 * j + 1]));
            w.y = relu_pack2(acc_add2(r[8 * j + 2], r[8 * j + 3], bv[8 * j + 2], bv[8 * j + 3]));
            w.z = relu_pack2(acc_add2(r[8 * j + 4], r[8 * j + 5], bv[8 * j + 4], bv[8 * j + 5]));
            w.w = relu_pack2(acc_add2(r[8 * j + 6], r[8 * j + 7], bv[8 * j + 6], bv[8 * j + 7]));
            const uint32_t chunk16 = (uint32_t)(eh * 4 + j);   // 16-byte chunk in the 128-byte row
            *reinterpret_cast<uint4*>(rowp + ((chunk16 ^ sw) << 4)) = w;
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&c1empty[buf]);                  // accumulator drained
          mbar_arrive(&a2full[buf]);                   // bf16 chunk staged for the second GEMM
        }
        chain_bar();
        if (issuer) {                                  // the same bytes are the O tile in HBM
          tma_store_2d(&tmO, dst, c * CH_BN, m0);
          tma_store_2d(&tmO, dst + CH_A_BYTES, c * CH_BN + CH_BK, m0);
          bulk_commit();
        }
      }
      // ---- T1 = relu(acc2 + b1), staged in sT.  Bulk groups retire in order:
      // with this tile's C O-chunk stores still allowed in flight, the previous
      // tile's T1 store has been read out of sT.
      mbar_wait(t2full, tt & 1);
      tc_fence_after();
      if (issuer) {
        if (C >= 4) bulk_wait_read<4>();
        else if (C == 3) bulk_wait_read<3>();
        else if (C == 2) bulk_wait_read<2>();
        else bulk_wait_read<1>();
      }
      chain_bar();
      for (int kb = 0; kb < a.N2 / 64; ++kb) {
        const int col = kb * 64 + eh * 32;
        uint32_t r[32];
        tmem_ld_32x32b_x32(tacc2 + ((uint32_t)(q * 32) << 16) + col, r);
        float bv[32];
        const float4* bp = reinterpret_cast<const float4*>(a.bias2 + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 b4 = __ldg(bp + j);
          bv[4 * j] = b4.x;
          bv[4 * j + 1] = b4.y;
          bv[4 * j + 2] = b4.z;
          bv[4 * j + 3] = b4.w;
        }
        tmem_wait_ld();
        uint8_t* rowp = sT + kb * CH_A_BYTES + row * 128;   // K block kb of T1
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 w;
          w.x = relu_pack2(acc_add2(r[8 * j + 0], r[8 * j + 1], bv[8 * j + 0], bv[8 * j + 1]));
          w.y = relu_pack2(acc_add2(r[8 * j + 2], r[8 * j + 3], bv[8 * j + 2], bv[8 * j + 3]));
          w.z = relu_pack2(acc_add2(r[8 * j + 4], r[8 * j + 5], bv[8 * j + 4], bv[8 * j + 5]));
          w.w = relu_pack2(acc_add2(r[8 * j + 6], r[8 * j + 7], bv[8 * j + 6], bv[8 * j + 7]));
          const uint32_t chunk16 = (uint32_t)(eh * 4 + j);
          *reinterpret_cast<uint4*>(rowp + ((chunk16 ^ sw) << 4)) = w;
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(t2empty);
      chain_bar();
      if (issuer) {
        for (int kb = 0; kb < a.N2 / 64; ++kb)
          tma_store_2d(&tmT, sT + kb * CH_A_BYTES, kb * CH_BK, m0);
        bulk_commit();
      }
    }
    if (issuer) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

static int chain_smem(const ChainArgs& a) {
  return 1024 + a.stages * CH_STAGE + 2 * CH_A2_BYTES + a.b2_stages * a.N2 * CH_BK * 2 +
         (a.N2 / 64) * CH_A_BYTES +
         8 * (2 * a.stages + 2 * a.b2_stages + 10) + 16;
}

bool chain_config(ChainArgs& a) {
  if (a.N1 % CH_BN != 0 || a.N2 % 64 != 0 || a.N2 < 64 || a.N2 > 256) return false;
  // the first GEMM's ring (A from HBM) needs the depth; two weight stages suffice
  for (a.stages = 8; a.stages >= 2; --a.stages)
    for (a.b2_stages = 3; a.b2_stages >= 2; --a.b2_stages)
      if (chain_smem(a) <= CH_SMEM_MAX) return true;
  return false;
}

cudaError_t chain_launch(const ChainArgs& a, const CUtensorMap& tA, const CUtensorMap& tB1,
                         const CUtensorMap& tR, const CUtensorMap& tI, const CUtensorMap& tB2,
                         const CUtensorMap& tO, const CUtensorMap& tT, int num_sms,
                         cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(chain_gemm_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, CH_SMEM_MAX);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = a.tiles_m < num_sms ? a.tiles_m : num_sms;
  return launch_pdl(chain_gemm_kernel, dim3(grid), dim3(CH_THREADS), chain_smem(a), st, tA, tB1,
                    tR, tI, tB2, tO, tT, a);
}

}  // namespace b2
