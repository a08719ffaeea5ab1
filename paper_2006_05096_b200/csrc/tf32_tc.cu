// fp32 plans on the tensor cores: 3xTF32 GEMM / implicit-GEMM conv (sm_100a).
//
//   D = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T      (kind::tf32, fp32 accumulate)
//
// (A_hi B_hi in one TMEM accumulator, the cross terms in another) with
// x_hi = x with its low 13 mantissa bits cleared (exactly representable
// in TF32) and x_lo = x - x_hi (exact in fp32; the MMA keeps its top 11
// bits).  The dropped A_lo B_lo term and the truncation of x_lo are ~2^-22
// relative, so results track an fp32 FFMA GEMM (the fp32 parity bound is 1e-4
// normwise against fp64) at tensor-core speed instead of the CUDA cores'.
//
// The tensor core's fp32 accumulation is not round-to-nearest per add (a
// single accumulator over K = 4608 drifted ~5e-5 normwise, measured), so the
// K loop is cut into chunks of F_KCHUNK K blocks: each chunk accumulates in a
// fresh TMEM buffer (double buffered) and the epilogue adds the chunk sums in
// fp32 registers (RN), bounding the per-accumulator add count independently
// of K.
//
// Weights are split once at plan creation (B_hi and B_lo tensors).  Activation
// tiles are split in shared memory: after TMA lands an fp32 A tile (128 rows x
// 32 fp32 = 128 B rows, 128B swizzle), four "splitter" warps rewrite it in
// place as A_hi and write A_lo next to it — same swizzled offsets, so both are
// valid UMMA operands — before the MMA warp consumes the stage.
//
// Warp roles: warp 0 TMA producer, warp 1 MMA issuer (converged, elected
// lane), warps 2..9 epilogue (fp32 out, bias / residual / activation, 16-byte
// stores), warps 10..13 splitters.  Tile 128 x 128, K block 32, TMEM double
// buffered.
#include "common.cuh"
#include "kernels.h"

namespace b2 {

constexpr int F_BM = 128, F_BN = 128, F_BK = 32;
constexpr int F_EPI_WARPS = 8, F_SPLIT_WARPS = 4;
constexpr int F_THREADS = (2 + F_EPI_WARPS + F_SPLIT_WARPS) * 32;
constexpr int F_A_BYTES = F_BM * F_BK * 4;        // 16 KB
constexpr int F_B_BYTES = F_BN * F_BK * 4;        // 16 KB
constexpr int F_STAGE = 2 * F_A_BYTES + 2 * F_B_BYTES;   // A_hi | A_lo | B_hi | B_lo
constexpr int F_STAGES = 3;
constexpr int F_KCHUNK = 1;                       // K blocks per TMEM partial sum
constexpr int F_SMEM = F_STAGES * F_STAGE + 1024 + 512;

B2_DEV float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__global__ void __launch_bounds__(F_THREADS, 1)
    tf32_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmBh,
                     const __grid_constant__ CUtensorMap tmBl, const TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + F_STAGES * F_STAGE);
  uint64_t* split = full + F_STAGES;     // A_hi / A_lo ready (128 splitter threads)
  uint64_t* empty = split + F_STAGES;
  uint64_t* tfull = empty + F_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_index_uniform();
  const int lane = threadIdx.x & 31;
  const int ntiles = a.tiles_m * a.tiles_n;
  const int KB = a.kblocks;                  // 32-wide K blocks

  if (threadIdx.x == 0) {
    for (int s = 0; s < F_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], F_SPLIT_WARPS * 32);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], F_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmBh);
    tma_prefetch_desc(&tmBl);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = uniform_u32(*tmem_slot);
  pdl_wait();
  pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int cpb = a.C / F_BK;            // im2col: 32-channel K blocks per filter tap
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t / a.tiles_n) * F_BM;
        const int n0 = (t % a.tiles_n) * F_BN;
        int iw0 = 0, ih0 = 0, img = 0;
        if (a.a_im2col) {
          img = m0 / a.OHW;
          const int rem = m0 - img * a.OHW;
          const int oh = rem / a.OW;
          ih0 = oh * a.stride - a.pad;
          iw0 = (rem - oh * a.OW) * a.stride - a.pad;
        }
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * F_STAGE;
          mbar_arrive_expect_tx(&full[stage], F_A_BYTES + 2 * F_B_BYTES);
          if (a.a_im2col) {
            const int tap = kb / cpb;
            const int c0 = (kb - tap * cpb) * F_BK;
            const int r = tap / a.S;
            const int s2 = tap - r * a.S;
            tma_load_im2col_4d(st, &tmA, &full[stage], c0, iw0, ih0, img, (uint16_t)s2,
                               (uint16_t)r);
          } else {
            tma_load_2d(st, &tmA, &full[stage], kb * F_BK, m0);
          }
          tma_load_2d(st + 2 * F_A_BYTES, &tmBh, &full[stage], kb * F_BK, n0);
          tma_load_2d(st + 2 * F_A_BYTES + F_B_BYTES, &tmBl, &full[stage], kb * F_BK, n0);
          if (++stage == F_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = make_idesc(F_BM, F_BN, 2u);   // TF32 x TF32 -> FP32
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;                                // partial-sum chunks issued by this CTA
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kc = 0; kc < KB; kc += F_KCHUNK, ++it) {
        const int as = it & 1;
        mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        // main product A_hi B_hi and the two small cross terms in separate
        // accumulators: the cross terms are ~2^-11 of the result, so their
        // accumulation error is negligible and the main one sees 4 adds per K block
        const uint32_t d = tmem_base + as * 2 * F_BN;
        const uint32_t dx = d + F_BN;
        const int kend = kc + F_KCHUNK < KB ? kc + F_KCHUNK : KB;
        for (int kb = kc; kb < kend; ++kb) {
          mbar_wait(&split[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * F_STAGE);
          const uint64_t ah = smem_desc_sw128(st);
          const uint64_t al = smem_desc_sw128(st + F_A_BYTES);
          const uint64_t bh = smem_desc_sw128(st + 2 * F_A_BYTES);
          const uint64_t bl = smem_desc_sw128(st + 2 * F_A_BYTES + F_B_BYTES);
#pragma unroll
          for (int k = 0; k < F_BK / 8; ++k) {   // K = 8 per tf32 UMMA (32 B)
            const uint32_t acc0 = (kb != kc || k != 0) ? 1u : 0u;
            if (elect_one()) umma_tf32(d, ah + 2 * k, bh + 2 * k, idesc, acc0);
            if (elect_one()) umma_tf32(dx, ah + 2 * k, bl + 2 * k, idesc, acc0);
            if (elect_one()) umma_tf32(dx, al + 2 * k, bh + 2 * k, idesc, 1u);
          }
          if (elect_one()) umma_commit(&empty[stage]);
          if (++stage == F_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit(&tfull[as]);
      }
    }
  } else if (warp < 2 + F_EPI_WARPS) {
    // ------------------------------------------------------------ epilogue (fp32 out)
    // thread = one tile row; columns eh*32 + {0, 64}; chunk partial sums are
    // added in registers, then bias / residual / activation, 16-byte stores
    const int lg = warp & 3;
    const int eh = (warp - 2) >> 2;
    float* outp = reinterpret_cast<float*>(a.out);
    const float* resp = reinterpret_cast<const float*>(a.res);
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int m0 = (t / a.tiles_n) * F_BM;
      const int n0 = (t % a.tiles_n) * F_BN;
      const int row = m0 + lg * 32 + lane;
      float acc[2][32];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[h][j] = 0.f;
      for (int kc = 0; kc < KB; kc += F_KCHUNK, ++it) {
        const int as = it & 1;
        mbar_wait(&tfull[as], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t(lg * 32) << 16) + as * 2 * F_BN + eh * 32;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t rm[32], rx[32];
          tmem_ld_32x32b_x32(taddr + h * 64, rm);
          tmem_ld_32x32b_x32(taddr + F_BN + h * 64, rx);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[h][j] += __uint_as_float(rm[j]) + __uint_as_float(rx[j]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[as]);
      }
      if (row < a.M) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col0 = n0 + eh * 32 + h * 64;
          if (col0 >= a.N) continue;
          float* v = acc[h];
          const bool full4 = col0 + 32 <= a.N && (a.N & 3) == 0;
          if (full4) {
            if (a.bias) {
              const float4* bp = reinterpret_cast<const float4*>(a.bias + col0);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 b4 = __ldg(bp + q);
                v[4 * q] += b4.x; v[4 * q + 1] += b4.y; v[4 * q + 2] += b4.z; v[4 * q + 3] += b4.w;
              }
            }
            if (resp) {
              const float4* rp = reinterpret_cast<const float4*>(resp + (size_t)row * a.ldres + col0);
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 r4 = __ldg(rp + q);
                v[4 * q] += r4.x; v[4 * q + 1] += r4.y; v[4 * q + 2] += r4.z; v[4 * q + 3] += r4.w;
              }
            }
            float4* op = reinterpret_cast<float4*>(outp + (size_t)row * a.ldo + col0);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              op[q] = make_float4(act_apply(v[4 * q], a.act), act_apply(v[4 * q + 1], a.act),
                                  act_apply(v[4 * q + 2], a.act), act_apply(v[4 * q + 3], a.act));
          } else {
            for (int j = 0; j < 32 && col0 + j < a.N; ++j) {
              float x = v[j];
              if (a.bias) x += a.bias[col0 + j];
              if (resp) x += resp[(size_t)row * a.ldres + col0 + j];
              outp[(size_t)row * a.ldo + col0 + j] = act_apply(x, a.act);
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ splitters
    // thread g rewrites A row g of each stage: hi in place, lo in the A_lo slot
    const int g = threadIdx.x - (2 + F_EPI_WARPS) * 32;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&full[stage], phase);
        float4* hi = reinterpret_cast<float4*>(smem + stage * F_STAGE + g * 128);
        float4* lo = reinterpret_cast<float4*>(smem + stage * F_STAGE + F_A_BYTES + g * 128);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {   // rotated per row: conflict-free 16-byte accesses
          const int j = (jj + g) & 7;
          const float4 x = hi[j];
          const float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
          hi[j] = h;
          lo[j] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
        }
        fence_proxy_async_smem();
        mbar_arrive(&split[stage]);
        if (++stage == F_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

cudaError_t tf32_gemm_launch(const TcArgs& a, const CUtensorMap& ta, const CUtensorMap& tbh,
                             const CUtensorMap& tbl, int num_sms, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(tf32_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int tiles = a.tiles_m * a.tiles_n;
  const int grid = tiles < num_sms ? tiles : num_sms;
  return launch_pdl(tf32_gemm_kernel, dim3(grid), dim3(F_THREADS), F_SMEM, st, ta, tbh, tbl, a);
}

}  // namespace b2
