// Kernel launch interfaces used by the executor (runtime.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace b2 {

// ---- tcgen05 GEMM / implicit-GEMM conv (bf16) -------------------------------
struct TcArgs {
  int M, N;
  int kblocks;          // ceil(K / 64)
  int Kreal;            // gather mode: R*S*C (chunks at k >= Kreal read as zero)
  const float* bias;    // [N] fp32 or nullptr
  const bf16* res;      // [M, ldres] or nullptr
  int ldres;
  bf16* out;            // [M, ldo]
  int ldo;
  int act;
  int tiles_m, tiles_n;
  // gather (implicit im2col) parameters, NHWC input
  const bf16* x;
  int H, W, C, OW, OHW, S, stride, pad;
  int R;
  int gmode;            // 1: C % 64 == 0 (one filter tap per K block)
                        // 2: S*C <= 64, C = 2^c_log2 (one filter row per K block)
                        // 3: generic (per-chunk tap decomposition)
  int c_log2, SC;
  int tma_epi;          // epilogue through smem + TMA store (N % 8 == 0, BN >= 64)
  int stages;           // smem pipeline depth (0 = the most that fits)
  int epi_debug;        // 0 normal; 1 drain TMEM only (no math/stores) — profiling aid
  int a_narrow;         // K <= 32 plain GEMM: A boxes 32 (SW64) or 16 (SW32) elements wide, not 64
  int ts_debug;         // B2_GEMM_TS=1: first/last CTA print phase timestamps — profiling aid
  int OH;               // s2d stems: output rows per image (M tile = one output row)
  int out3d;            // output TMA map is [rows, OW, C]: box rows clip at OW
  int a_im2col;         // A via TMA: 3 = space-to-depth stem (one output row per M tile,
                        //     tiled 4D view with overlapping pixel stride, K block = filter row);
                        // 1 = 64-channel im2col boxes (C % 64 == 0, 128B swizzle);
                        // 2 = one 8-channel filter tap per 2 KB box (C == 8 stems), 8 taps
                        //     per K block in the non-swizzled K-major layout
  int reverse;          // walk M tiles last-to-first (L2 reuse across layers)
  int nsplit;           // split-K factor (1 = none): partials red.add'ed into ws
  float* ws;            // split-K fp32 partials [nsplit][M][N]
  int fold_kind;        // extra K blocks: 0 residual x identity; 1 shortcut x (stride 1, 2D)
                        // against its weights; 2 strided shortcut x (im2col TMA)
  int ds_H, ds_W;       // fold_kind 2: shortcut input geometry (uses OW, OHW, stride too)
  int res_kblocks;      // >0: residual folded into the MMA as [A | res] x [W | I]^T;
                        // BN/64 extra K blocks per tile, A from tmR, B from the identity
};

// ---- banded implicit-GEMM conv (conv_band.cu) --------------------------------
struct BandArgs {
  int B, H, W, N;       // output NHWC [B, H, W, N]
  int Wp;               // A view row pitch in pixels (W + S - 1, or the s2d width)
  int R, S;             // taps; tap (r, s) reads A row p + r * Wp + s
  int CG;               // channel groups per tap (C / 64; 1 for the s2d stem)
  int x0, y0;           // A box start offsets (-pad for zero-filled halos)
  int kblocks;          // Kpad / 64 (weight K blocks)
  int tiles_n;          // N / BN
  int nseg, seg_w;      // column segments (rows wider than one band pitch): valid output
                        // columns per segment (the last one takes the rest)
  // geometry chosen by band_config
  int bh, nbands, MT;
  int a_box_bytes, a_stage_bytes, a_stages, b_stages, b_resident, tmem_cols;
  int pair;             // CTA-pair kernel (N = 64, resident weights): M = 256 UMMAs over two bands
  int pool2;            // fused 2x2/2 max-pool epilogue (Wp == 128: one output row per M tile)
  const float* bias;
  bf16* out;
  int act;
  // fused 3x3/s2/p1 max-pool epilogue (stem_pool_kernel): pooled output
  bf16* pout;
  int PH, PW;
};
bool band_config(BandArgs& a, int bn, int cgw, int mt_cap = 4);
bool band_supported(const BandArgs& a, int bn, int cgw, int act);
int band_smem_bytes(const BandArgs& a, int bn);
bool stem_pool_config(BandArgs& a);
cudaError_t stem_pool_launch(const BandArgs& a, const CUtensorMap& ta, const CUtensorMap& tb,
                             int num_sms, cudaStream_t st);
cudaError_t conv_band_launch(const BandArgs& a, int bn, int cgw, const CUtensorMap& ta,
                             const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& to2,
                             int num_sms, cudaStream_t st);

// ---- chained 1x1 convs (chain_tc.cu): block tail conv -> next block's conv1 --
struct ChainArgs {
  int M, N1, N2;        // O = relu(A W3^T + b1 + fold) [M, N1]; T1 = relu(O W1^T + b2) [M, N2]
  int kblocks;          // K1 / 64
  int res_kblocks;      // fold K blocks per 128-column O chunk
  int fold_kind;        // 0 residual x identity; 1 shortcut x (2D); 2 strided shortcut (im2col)
  int OW, OHW, stride;  // fold_kind 2 geometry
  int tiles_m, reverse;
  int stages, b2_stages;   // set by chain_config
  const float* bias1;
  const float* bias2;
};
bool chain_config(ChainArgs& a);
cudaError_t chain_launch(const ChainArgs& a, const CUtensorMap& tA, const CUtensorMap& tB1,
                         const CUtensorMap& tR, const CUtensorMap& tI, const CUtensorMap& tB2,
                         const CUtensorMap& tO, const CUtensorMap& tT, int num_sms,
                         cudaStream_t st);

int tc_pick_bn(long M, int N, int num_sms);
// BN and single-CTA vs CTA-pair kernel from the per-SM clock model (gemm_tc.cu)
int tc_pick_config(long M, int N, int kblocks, bool res_fold, int num_sms, bool pair_allowed,
                   bool* pair_out);
cudaError_t tf32_gemm_launch(const TcArgs& a, const CUtensorMap& ta, const CUtensorMap& tbh,
                             const CUtensorMap& tbl, int num_sms, cudaStream_t st);
int tc_pick_split(long tiles, int kt, int num_sms);
cudaError_t splitk_finalize(const float* ws, int nsplit, const float* bias, const bf16* res,
                            bf16* out, long M, int N, int act, cudaStream_t st);
int tc2_pick_bn(long M, int N, int num_sms);
cudaError_t tc_gemm2_launch(const TcArgs& a, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                            const CUtensorMap& to, const CUtensorMap& tr, const CUtensorMap& ti,
                            int num_sms, cudaStream_t st);
cudaError_t tc_gemm_launch(const TcArgs& a, int bn, bool gather, const CUtensorMap& ta,
                           const CUtensorMap& tb, const CUtensorMap& to, const CUtensorMap& tr,
                           const CUtensorMap& ti, int num_sms, cudaStream_t st);

cudaError_t attention_tc(const CUtensorMap& tm_qkv, bf16* out, int B, int H,
                         const uint32_t* keymask, cudaStream_t st);

// ---- SIMT kernels (templated on storage type: float or bf16) -----------------
struct GemmSimtArgs {
  int M, N, K;          // K = real reduction length
  const void* a;        // activations (T)
  int lda;              // linear mode: row stride of A (elements)
  const void* w;        // weights [N, ldw] (T)
  int ldw;
  const float* bias;
  const void* res;      // [M, N] (T) or nullptr
  void* out;            // [M, N] (T)
  int act;
  int conv;             // 1: implicit im2col gather from NHWC x
  int H, W, C, OW, OHW, S, stride, pad;
};

// fused INPUT -> LINEAR(act) -> LINEAR(act) -> OUTPUT for small MLPs (kernels.cu)
struct MlpArgs {
  const float* in;              // fp32 input [B][K1]
  const void* w1; const void* w1lo;   // [N1][ldw1] (T); lo part of a 3xTF32 split or nullptr
  int ldw1;
  const float* b1;
  int act1;
  const void* w2; const void* w2lo;
  int ldw2;
  const float* b2;
  int act2;
  void* xin;                    // input tensor [B][K1] (T): the packed input, for read-back
  void* h;                      // hidden tensor [B][N1] (T)
  void* y;                      // logits tensor [B][N2] (T)
  float* out;                   // plan output [B][out_stride], this tensor at out_off
  long out_stride, out_off;
  int B, K1, N1, N2;
  unsigned* counters;           // per 16-row group, zero between launches
};
template <typename T> cudaError_t mlp2(const MlpArgs& a, cudaStream_t st);
// im2col rows of an NHWC fp32 conv input: col[m][k], k = (r, s, c) < R*S*C, zero
// for k >= R*S*C up to kpad (the gathered 3xTF32 path for few-channel convs)
cudaError_t im2col_f32(const float* x, float* col, int B, int H, int W, int C, int R, int S,
                       int stride, int pad, int OH, int OW, int kpad, cudaStream_t st);
template <typename T> cudaError_t gemm_simt(const GemmSimtArgs& a, cudaStream_t st);
template <typename T>
cudaError_t input_pack(const float* in, T* out, int B, int C, int H, int W, int Cp,
                       cudaStream_t st);
cudaError_t input_pack_s2d(const float* in, bf16* out, int B, int C, int H, int W, int shift,
                           int H2, int W2, cudaStream_t st);
cudaError_t tokens_pack(const int64_t* in, int32_t* out, uint32_t* mask, int B, int S,
                        int stride, int vocab, cudaStream_t st);
template <typename T>
cudaError_t dwconv(const T* x, const T* w_rsc, const float* bias, T* y, int B, int H, int W,
                   int C, int R, int stride, int pad, int OH, int OW, int act, cudaStream_t st);
template <typename T>
cudaError_t maxpool(const T* x, T* y, int B, int H, int W, int C, int k, int stride, int pad,
                    int OH, int OW, cudaStream_t st);
template <typename T>
cudaError_t avgpool(const T* x, T* y, int B, int HW, int C, cudaStream_t st);
template <typename T>
cudaError_t layernorm(const T* x, const T* res, const float* g, const float* b, T* y, long rows,
                      int D, float eps, cudaStream_t st);
template <typename T>
cudaError_t embed_ln(const int32_t* ids, const T* word, const T* pos, const T* type,
                     const float* g, const float* b, T* y, int B, int S, int D, float eps,
                     cudaStream_t st);
template <typename T>
cudaError_t attention(const T* qkv, T* out, int B, int S, int H, int Dh,
                      const uint32_t* keymask, cudaStream_t st);
template <typename T>
cudaError_t act_ew(const T* x, T* y, long n, int act, cudaStream_t st);
template <typename T>
cudaError_t output_gather(const T* src, float* out, int B, long elems, long out_stride,
                          long offset, cudaStream_t st);
cudaError_t gen_normal(float* out, long n, uint64_t seed, cudaStream_t st);
cudaError_t gen_tokens(int64_t* out, long n, int S, int stride, int vocab, uint64_t seed,
                       cudaStream_t st);
cudaError_t flush_l2(void* buf, size_t bytes, cudaStream_t st);

template <typename T>
cudaError_t convert_f32(const float* src, T* dst, long n, cudaStream_t st);

}  // namespace b2
