// libb2 executor: b200-plan parsing, weight upload in kernel layouts, per-batch
// activation workspaces, CUDA-graph replay, and the device-timed closed-loop
// measurement that replaces the reference profiler's host RPC timing loop
// (pkg/src/modelci/profiler/clients.py:161-255).  C ABI in include/b2.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <chrono>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/b2.h"
#include "common.cuh"
#include "kernels.h"

// NVTX ranges around the timed regions (bench / forward_host) and around each
// op of the eager profile pass, so a profiler (ncu --nvtx, nsys) attributes
// kernels to the profiling cell that launched them.  Header-only NVTX3: free
// unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* fmt, ...) {
    char buf[96];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

static bool g_pdl = true;   // B2_PDL=0 -> plain stream-ordered launches
bool pdl_enabled() { return g_pdl; }

namespace {

using namespace b2;

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(B2_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),   \
                  __FILE__, __LINE__);                                                    \
  } while (0)

// ------------------------------------------------------------------ plan format
enum {
  OP_INPUT = 1, OP_TOKENS = 2, OP_CONV = 3, OP_LINEAR = 4, OP_DWCONV = 5, OP_MAXPOOL = 6,
  OP_AVGPOOL = 7, OP_LAYERNORM = 8, OP_EMBED = 9, OP_ATTENTION = 10, OP_OUTPUT = 11, OP_ACT = 12
};
constexpr int NPARAM = 31;

#pragma pack(push, 1)
struct Header {
  char magic[4];
  uint32_t version, dtype, n_tensors, n_weights, n_ops, input_kind, in_elems, out_elems,
      meta_len, r0, r1;
};
struct TensorRec {
  uint32_t kind, elems;
  int32_t shape[4];
};
struct WeightRec {
  uint64_t offset, numel;
  int32_t shape[4];
};
struct OpRec {
  uint32_t kind;
  int32_t p[NPARAM];
};
#pragma pack(pop)
static_assert(sizeof(Header) == 48, "header");
static_assert(sizeof(TensorRec) == 24, "tensor rec");
static_assert(sizeof(WeightRec) == 32, "weight rec");
static_assert(sizeof(OpRec) == 128, "op rec");

// CRC-32 (IEEE, reflected), slice-by-8: ~8x the byte-table loop, which
// cost ~0.5 s of plan creation on the 436 MB BERT blob.
uint32_t crc32(const uint8_t* p, size_t n) {
  static uint32_t table[8][256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int s = 1; s < 8; ++s) table[s][i] = (table[s - 1][i] >> 8) ^ table[0][table[s - 1][i] & 0xFF];
    init = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint32_t lo, hi;
    memcpy(&lo, p + i, 4);
    memcpy(&hi, p + i + 4, 4);
    lo ^= c;
    c = table[7][lo & 0xFF] ^ table[6][(lo >> 8) & 0xFF] ^ table[5][(lo >> 16) & 0xFF] ^
        table[4][lo >> 24] ^ table[3][hi & 0xFF] ^ table[2][(hi >> 8) & 0xFF] ^
        table[1][(hi >> 16) & 0xFF] ^ table[0][hi >> 24];
  }
  for (; i < n; ++i) c = table[0][(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// ------------------------------------------------------------------ TMA maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// bf16 matrix [rows, cols] with a row pitch in bytes; box = 64 cols x box_rows,
// 128-byte swizzle (the canonical UMMA K-major layout)
bool make_tmap_bf16(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                    uint64_t row_bytes, uint32_t box_rows, uint32_t box_cols = 64,
                    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 matrix [rows, cols] with row pitch in bytes; box = 32 cols (128 B) x
// box_rows, 128-byte swizzle (the 3xTF32 GEMM's K-major operand layout)
bool make_tmap_f32(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t row_bytes, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                   cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  }
  return fn;
}

// NHWC bf16 activation [N, H, W, C] for implicit-GEMM conv A tiles: 128 output
// pixels x 64 channels per load, filter offsets supplied per load
bool make_tmap_im2col(CUtensorMap* m, const void* base, int N, int H, int W, int C, int R, int S,
                      int stride, int pad, int cpp, int esize = 2) {
  EncodeIm2colFn fn = encode_im2col_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C * esize, (cuuint64_t)W * C * esize,
                           (cuuint64_t)H * W * C * esize};
  int lower[2] = {-pad, -pad};
  int upper[2] = {pad - (S - 1), pad - (R - 1)};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  if (fn(m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
         const_cast<void*>(base), dims, strides, lower, upper, (cuuint32_t)cpp, 128, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE,
         cpp * esize == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  const int esz_total = esize;
  (void)esz_total;
  // driver <= 13.1 workaround for tensors under 128 KB (mirrors CUTLASS)
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && (uint64_t)N * H * W * C * esize < 131072)
    reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
  return true;
}

// ------------------------------------------------------------------ executor state
struct Layer {
  int kind;
  int p[NPARAM];
  // device parameters
  void* w = nullptr;        // main weight in kernel layout (T)
  float* bias = nullptr;    // fp32
  float* g = nullptr;       // LayerNorm gamma (fp32)
  float* b = nullptr;       // LayerNorm beta (fp32)
  void* w2 = nullptr;       // embed: pos table (T)
  void* w3 = nullptr;       // embed: type row (T)
  // GEMM execution choices
  bool tc = false, gather = false;
  bool im2col = false;      // A via TMA im2col (C % 64 == 0 convs, or C == 8 stems)
  // space-to-depth stem (conv) / producer (input): stride-2 conv on <= 4 real
  // channels re-expressed as a stride-1 conv on a 2x2 space-to-depth tensor
  bool s2d = false;
  int s2d_shift = 0, s2d_H2 = 0, s2d_W2 = 0, s2d_Rp = 0, s2d_creal = 0;
  int im2col_mode = 0;      // TcArgs::a_im2col
  int pool_op = -1;         // s2d stem: index of the 3x3/s2 max-pool fused into its epilogue
  int pool2_op = -1;        // band conv: index of the 2x2/s2 max-pool fused into its epilogue
  int ds_op = -1;           // 1x1 conv: index of the projection shortcut folded into its K loop
  int chain_op = -1;        // block-tail 1x1 conv: next block's 1x1 conv computed in the same kernel
  bool tf32 = false;        // fp32 plan conv/linear on the 3xTF32 tcgen05 GEMM (w = hi, w2 = lo)
  bool tf32_gather = false; // ... with its im2col A materialised first (convs with C % 32 != 0:
                            // the 3-channel stems), [M][kpad] fp32 in BatchState::col
  bool band8 = false;       // 3x3/s1 conv on an 8-channel padded image: conv_band CGW = 8,
                            // weights [N][r][4][8] (paired taps, 4th tap zero)
  bool fused = false;       // max-pool executed inside its producer (no launch)
  int gmode = 0;            // see TcArgs::gmode
  int K = 0, kpad = 0, ldw = 0;
};

struct BatchState {
  int batch = 0;
  std::vector<void*> act;          // per tensor (slices of arena)
  void* arena = nullptr;
  void* d_in = nullptr;            // internal input buffer
  float* d_out = nullptr;          // internal output buffer
  std::vector<int> bn;             // per layer (tc)
  std::vector<CUtensorMap> tmA;    // per layer (tc, TMA mode)
  std::vector<CUtensorMap> tmB;    // per layer (tc): weights, box rows = BN
  std::vector<CUtensorMap> tmO;    // per layer (tc): output, 32x32 box, 64B swizzle
  std::vector<CUtensorMap> tmR;    // per layer (tc, residual fold): residual as an A operand
  std::vector<char> fold;          // per layer: residual folded into the MMA
  unsigned* mlp_ctr = nullptr;     // fused MLP: per-16-row-group arrival counters
  float* col = nullptr;            // gathered 3xTF32 convs: im2col A [M][kpad] fp32 (shared)
  std::vector<char> a_narrow;      // per layer: A box width for K <= 32 (0 = 64)
  std::vector<CUtensorMap> tmI;    // per layer: identity [256 x 256] (box rows = BN) for the fold
  std::vector<char> band;          // per layer: banded implicit-GEMM conv (conv_band.cu)
  std::vector<char> pair;          // per layer: CTA-pair GEMM (tc_gemm2_kernel)
  std::vector<char> chain;         // per layer: chained with the next conv1 (chain_tc.cu)
  std::vector<int> split;          // per layer: split-K factor (small batches)
  float* ws = nullptr;             // split-K fp32 partial slices (shared by the layers)
  std::vector<ChainArgs> cargs;
  std::vector<CUtensorMap> tmB2, tmT;   // chain: second weights, second output
  std::vector<BandArgs> bargs;     // per layer (band): geometry chosen by band_config
  cudaGraphExec_t graph = nullptr;
  void* h_in = nullptr;            // pinned (e2e)
  void* h_out = nullptr;
  // e2e pipelining: a second input/output buffer pair and its graph, so the
  // H2D of step i+1 and the D2H of step i-1 overlap the forward of step i
  void* d_in2 = nullptr;
  float* d_out2 = nullptr;
  void* h_out2 = nullptr;
  cudaGraphExec_t graph2 = nullptr;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
};

}  // namespace

struct b2_plan {
  int dtype = 1;
  int device = 0;
  int num_sms = 148;
  int input_kind = 0;
  long in_elems = 0, out_elems = 0;
  int vocab = 0;
  int seq = 0;               // tokens per sample (TOKENS op)
  double flops = 0, weight_bytes = 0;
  std::vector<TensorRec> tensors;
  std::vector<Layer> layers;
  std::vector<char> virt;    // per tensor: fused away (never materialised)
  std::vector<void*> allocs;
  std::map<int, BatchState> states;
  cudaStream_t stream = nullptr;
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  bool force_simt = false;
  int launches = 0;
  int epi_mode = 0;          // B2_EPI_MODE: 0 TMA-store epilogue, 1 drain-only, 2 direct stores
  int fold_max_k = 1024;     // B2_FOLD_MAX_K: fold residuals into the MMA when K <= this
  bool use_im2col = true;    // B2_IM2COL=0 -> cp.async gather for C % 64 == 0 convs
  bool use_s2d = true;       // B2_S2D=0 -> stems on the cp.async gather path
  bool im2col8 = false;      // B2_IM2COL8=1 -> 8-channel-tap im2col TMA for C == 8 stems
                             // (correct, but issue-bound on 2 KB boxes: slower than gather)
  bool use_band = true;      // B2_BAND=0 -> stride-1 k x k convs and s2d stems on gemm_tc
  bool use_pair = true;      // B2_PAIR=0 -> single-CTA tc_gemm only
  bool band_pair = true;     // B2_BAND_PAIR=0 -> single-CTA band kernel for N = 64
  bool narrow_k = true;      // B2_NARROW_K=0 -> 64-wide A boxes for K <= 32 too
  bool verbose = false;      // B2_VERBOSE=1: per-layer kernel choices on stderr
  long pair_min_m = 4096;    // B2_PAIR_MIN_M: smallest M sent to the CTA-pair GEMM
  int pair_min_k = 0;        // B2_PAIR_MIN_K: shortest K sent to the CTA-pair GEMM
  bool use_pool_fusion = true;   // B2_POOL_FUSION=0 -> stem and max-pool as two kernels
  bool use_tf32 = true;          // B2_TF32=0 -> fp32 plans on the CUDA-core FFMA GEMM
  bool tf32_gather = true;       // B2_TF32_GATHER=0 -> few-channel fp32 convs on the FFMA GEMM
  bool use_ds_fold = true;       // B2_DS_FOLD=0 -> projection shortcuts as their own kernels
  bool alt_order = true;         // B2_ALT_ORDER=0 -> every GEMM walks M tiles forward
  bool use_split = true;         // B2_SPLIT=0 -> no split-K at small batch
  bool use_chain = true;         // B2_CHAIN=0 -> block-tail and next conv1 as two GEMMs
  bool chain_ds2 = false;        // B2_CHAIN_DS2=1 -> chain tails with a strided shortcut too
                                 // (measured: -13 us on ResNet-50 b=256 without)
  bool use_mlp_fusion = true;    // B2_MLP_FUSE=0 -> the toy MLP as pack + 2 GEMMs + gather
  int mlp_in = -1, mlp_l1 = -1, mlp_l2 = -1, mlp_out = -1;   // fused 2-layer MLP (plan_fuse_mlp)
  int band_max_n = 128;      // B2_BAND_MAX_N: widest conv (output channels) sent to conv_band
  void* identity = nullptr;  // bf16 I[256][256]
  void* stage = nullptr;     // weight-upload staging (plan creation only)
  size_t stage_bytes = 0;
  size_t dev_bytes = 0;      // device memory held (weights, arenas, I/O buffers; b2_plan_memory)
  float* zero_bias = nullptr;  // fp32 zeros[8192]: bias of bias-free layers in fused epilogues
  int stages_override = 0;   // B2_STAGES
  int ts_debug = 0;          // B2_GEMM_TS
  int force_bn = 0;          // B2_FORCE_BN
};

namespace {

template <typename T> size_t tsize() { return sizeof(T); }

// every plan-lifetime device allocation goes through here (b2_plan_memory)
cudaError_t dmalloc(b2_plan* pl, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess) pl->dev_bytes += bytes;
  return e;
}

int upload_f32(b2_plan* pl, const float* src, size_t n, float** out) {
  float* d = nullptr;
  const size_t padded = (n + 255) / 256 * 256;   // epilogues read whole 32-column chunks
  CK(dmalloc(pl, (void**)&d, padded * sizeof(float)));
  CK(cudaMemset(d, 0, padded * sizeof(float)));
  pl->allocs.push_back(d);
  CK(cudaMemcpy(d, src, n * sizeof(float), cudaMemcpyHostToDevice));
  pl->weight_bytes += n * sizeof(float);
  *out = d;
  return B2_OK;
}

// host fp32 -> device T via a plan-lifetime fp32 staging buffer and a
// conversion kernel on the legacy stream (the next synchronous cudaMemcpy
// into the staging buffer is ordered after it); freed once all weights are
// up.  Per-weight cudaMalloc/cudaFree/cudaDeviceSynchronize of the staging
// buffer cost seconds of worker start-up on BERT / VGG.
template <typename T> int upload_as(b2_plan* pl, const std::vector<float>& h, void** out) {
  const size_t need = h.size() * sizeof(float) + 16;
  if (need > pl->stage_bytes) {
    if (pl->stage) {
      CK(cudaDeviceSynchronize());
      CK(cudaFree(pl->stage));
    }
    CK(cudaMalloc(&pl->stage, need));
    pl->stage_bytes = need;
  }
  CK(cudaMemcpy(pl->stage, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  T* d = nullptr;
  CK(dmalloc(pl, (void**)&d, h.size() * sizeof(T) + 16));
  pl->allocs.push_back(d);
  CK(convert_f32<T>(static_cast<const float*>(pl->stage), d, (long)h.size(), 0));
  pl->weight_bytes += h.size() * sizeof(T);
  *out = d;
  return B2_OK;
}

// Find stride-2 stems fed directly by the INPUT op (<= 4 real channels, odd
// square filter, "same" padding, even H/W, one output row fits an M tile) and
// switch them and their INPUT op to the space-to-depth layout.
void plan_s2d(b2_plan* pl) {
  if (pl->dtype != B2_DT_BF16 || pl->force_simt || !pl->use_s2d) return;
  for (size_t ci = 0; ci < pl->layers.size(); ++ci) {
    Layer& Lc = pl->layers[ci];
    if (Lc.kind != OP_CONV) continue;
    const int* p = Lc.p;
    const int R = p[8], S = p[9], stride = p[10], pad = p[11];
    if (stride != 2 || R != S || (R & 1) == 0 || pad != (R - 1) / 2 || (p[4] & 1) ||
        (p[5] & 1) || p[13] > 128 || p[15] >= 0)
      continue;
    int in_op = -1, consumers = 0;
    for (size_t j = 0; j < pl->layers.size(); ++j) {
      const Layer& Lj = pl->layers[j];
      if (Lj.kind == OP_INPUT && Lj.p[0] == p[0]) in_op = (int)j;
      if (Lj.kind == OP_OUTPUT) {
        for (int q = 0; q < Lj.p[0]; ++q) consumers += Lj.p[1 + 2 * q] == p[0];
      } else if (Lj.kind != OP_INPUT && Lj.p[0] == p[0]) {
        ++consumers;
      } else if ((Lj.kind == OP_CONV && Lj.p[15] == p[0]) ||
                 ((Lj.kind == OP_LINEAR) && Lj.p[8] == p[0]) ||
                 (Lj.kind == OP_LAYERNORM && Lj.p[7] == p[0])) {
        ++consumers;
      }
    }
    if (in_op < 0 || consumers != 1) continue;
    Layer& Li = pl->layers[in_op];
    if (Li.p[1] > 4 || Li.p[4] != p[6]) continue;
    const int Rp = R / 2 + 1;
    for (Layer* L : {&Lc, &Li}) {
      L->s2d = true;
      L->s2d_shift = pad + 1;
      L->s2d_Rp = Rp;
      L->s2d_H2 = p[12] + Rp - 1;
      L->s2d_W2 = p[13] + 3;
      L->s2d_creal = Li.p[1];
    }
  }
}

// Fuse the 3x3 / stride-2 / pad-1 max-pool that is the only consumer of a
// ReLU space-to-depth stem into the stem's epilogue (conv_band.cu,
// stem_pool_kernel).  The stem's own output tensor is then never written.
void plan_fuse_pool(b2_plan* pl) {
  pl->virt.assign(pl->tensors.size(), 0);
  if (!pl->use_band || !pl->use_pool_fusion) return;
  for (size_t ci = 0; ci < pl->layers.size(); ++ci) {
    Layer& Lc = pl->layers[ci];
    if (Lc.kind != OP_CONV || !Lc.s2d || Lc.p[14] != ACT_RELU || Lc.p[7] != 64) continue;
    const int t = Lc.p[1];
    int pool = -1, users = 0;
    for (size_t j = 0; j < pl->layers.size(); ++j) {
      const Layer& Lj = pl->layers[j];
      if (j == ci) continue;
      bool uses = false;
      if (Lj.kind == OP_OUTPUT) {
        for (int q = 0; q < Lj.p[0]; ++q) uses |= Lj.p[1 + 2 * q] == t;
      } else if (Lj.kind != OP_INPUT && Lj.kind != OP_TOKENS) {
        uses = Lj.p[0] == t || (Lj.kind == OP_CONV && Lj.p[15] == t) ||
               (Lj.kind == OP_LINEAR && Lj.p[8] == t) || (Lj.kind == OP_LAYERNORM && Lj.p[7] == t);
      }
      if (uses) {
        ++users;
        if (Lj.kind == OP_MAXPOOL && Lj.p[0] == t) pool = (int)j;
      }
    }
    if (users != 1 || pool < 0) continue;
    const int* q = pl->layers[pool].p;   // in, out, H, W, C, k, stride, pad, OH, OW
    if (q[5] != 3 || q[6] != 2 || q[7] != 1 || q[2] != Lc.p[12] || q[3] != Lc.p[13] ||
        q[8] * 2 != q[2] || q[9] * 2 != q[3])
      continue;
    Lc.pool_op = pool;
    pl->layers[pool].fused = true;
    pl->virt[t] = 1;
  }
  // 3x3/1 band convs (VGG) followed by a 2x2/2 max-pool that is their only
  // consumer: the band epilogue pools row pairs / column pairs and writes only
  // the pooled tensor (needs one output row per M tile: band pitch 128).
  // N = 128 (streamed weights; VGG conv2_2 + pool2 0.811 + 0.237 -> 0.795 ms)
  // pairs rows inside a band; N = 64 keeps its resident weights with one-row
  // bands and pairs rows across consecutive units of a CTA (an even band
  // height pushed the weights out of shared memory: conv1_2 1.06 -> 1.64 ms).
  for (size_t ci = 0; ci < pl->layers.size() && pl->dtype == B2_DT_BF16; ++ci) {
    Layer& Lc = pl->layers[ci];
    const int* p = Lc.p;
    if (Lc.kind != OP_CONV || Lc.s2d || Lc.pool_op >= 0 || p[14] != ACT_RELU || p[15] >= 0 ||
        p[8] != 3 || p[9] != 3 || p[10] != 1 || p[11] != 1 || p[6] % 64 != 0 ||
        !(p[7] == 64 || p[7] == 128) || p[7] > pl->band_max_n || p[12] != p[4] ||
        p[13] != p[5] || (p[12] & 1) || (p[13] & 1) || p[13] + 2 <= 96 || p[13] > 2 * 126)
      continue;
    const int t = p[1];
    int pool = -1, users = 0;
    for (size_t j = 0; j < pl->layers.size(); ++j) {
      const Layer& Lj = pl->layers[j];
      if (j == ci) continue;
      bool uses = false;
      if (Lj.kind == OP_OUTPUT) {
        for (int q = 0; q < Lj.p[0]; ++q) uses |= Lj.p[1 + 2 * q] == t;
      } else if (Lj.kind != OP_INPUT && Lj.kind != OP_TOKENS) {
        uses = Lj.p[0] == t || (Lj.kind == OP_CONV && Lj.p[15] == t) ||
               (Lj.kind == OP_LINEAR && Lj.p[8] == t) || (Lj.kind == OP_LAYERNORM && Lj.p[7] == t);
      }
      if (uses) {
        ++users;
        if (Lj.kind == OP_MAXPOOL && Lj.p[0] == t) pool = (int)j;
      }
    }
    if (users != 1 || pool < 0) continue;
    const int* q = pl->layers[pool].p;   // in, out, H, W, C, k, stride, pad, OH, OW
    if (q[5] != 2 || q[6] != 2 || q[7] != 0 || q[8] * 2 != p[12] || q[9] * 2 != p[13]) continue;
    Lc.pool2_op = pool;
    pl->layers[pool].fused = true;
    pl->virt[t] = 1;
  }
}

// Fold a ResNet projection shortcut into the block's last 1x1 conv:
//   out = act(t2 W3^T + b3 + x Wd^T + bd)
// computed as one GEMM over K = [t2 | x (strided)] with B = [W3 | Wd], so the
// shortcut's output (411 MB at layer1, b=256) is neither written nor read
// back as a residual, and its kernel disappears.  Conditions: the shortcut
// is a plain 1x1 conv (pad 0, stride 1 or 2, no activation/residual) whose
// output feeds only this conv's residual input, channels multiples of 64.
void plan_fold_downsample(b2_plan* pl) {
  if (pl->dtype != B2_DT_BF16 || pl->force_simt || !pl->use_ds_fold) return;
  auto users = [&](int t) {
    int n = 0;
    for (const Layer& Lj : pl->layers) {
      if (Lj.kind == OP_OUTPUT) {
        for (int q = 0; q < Lj.p[0]; ++q) n += Lj.p[1 + 2 * q] == t;
      } else if (Lj.kind != OP_INPUT && Lj.kind != OP_TOKENS) {
        n += Lj.p[0] == t;
        n += (Lj.kind == OP_CONV && Lj.p[15] == t) || (Lj.kind == OP_LINEAR && Lj.p[8] == t) ||
             (Lj.kind == OP_LAYERNORM && Lj.p[7] == t);
      }
    }
    return n;
  };
  for (size_t ci = 0; ci < pl->layers.size(); ++ci) {
    Layer& C3 = pl->layers[ci];
    const int* p = C3.p;
    if (C3.kind != OP_CONV || p[15] < 0 || p[8] != 1 || p[9] != 1 || p[10] != 1 || p[11] != 0 ||
        p[7] % 64 != 0 || p[6] % 64 != 0)
      continue;
    for (size_t di = 0; di < pl->layers.size(); ++di) {
      Layer& D = pl->layers[di];
      const int* q = D.p;
      if (di == ci || D.kind != OP_CONV || q[1] != p[15] || q[8] != 1 || q[9] != 1 || q[11] != 0 ||
          (q[10] != 1 && q[10] != 2) || q[14] != ACT_NONE || q[15] >= 0 || q[6] % 64 != 0 ||
          q[7] != p[7] || q[12] != p[12] || q[13] != p[13] || users(p[15]) != 1)
        continue;
      C3.ds_op = (int)di;
      D.fused = true;
      pl->virt[p[15]] = 1;
      break;
    }
  }
}

// Chain a block's last 1x1 conv (O = relu(t2 W3^T + b3 + residual or folded
// shortcut)) with the next block's first 1x1 conv (T1 = relu(O W1^T + b1)) in
// one kernel (chain_tc.cu): O is written once and consumed from shared
// memory.  Needs 128 | N1, 64 | N2 <= 256.
void plan_chain(b2_plan* pl) {
  if (pl->dtype != B2_DT_BF16 || pl->force_simt || !pl->use_chain) return;
  for (size_t ci = 0; ci < pl->layers.size(); ++ci) {
    Layer& C3 = pl->layers[ci];
    const int* p = C3.p;
    if (C3.kind != OP_CONV || C3.fused || p[15] < 0 || p[8] != 1 || p[9] != 1 || p[10] != 1 ||
        p[11] != 0 || p[14] != ACT_RELU || p[6] % 64 != 0 || p[7] % 128 != 0)
      continue;
    for (size_t j = ci + 1; j < pl->layers.size(); ++j) {
      Layer& C1 = pl->layers[j];
      const int* q = C1.p;
      if (C1.kind != OP_CONV || C1.fused || q[0] != p[1] || q[8] != 1 || q[9] != 1 || q[10] != 1 ||
          q[11] != 0 || q[14] != ACT_RELU || q[15] >= 0 || q[7] % 64 != 0 || q[7] > 256 ||
          q[6] != p[7])
        continue;
      // measured (ResNet-50 b=256, per-op events): the chain wins where both
      // GEMMs are HBM-bound (N1 = 256: -30 us per block; N1 = 512 with
      // N2 = 128: -8..-22 us) and loses once they are operand-bound (N1 = 1024:
      // +24..+89 us — every 128-column chunk re-reads its A panel)
      if (!(p[7] <= 256 || (p[7] <= 512 && q[7] <= 128))) break;
      // a folded *strided* shortcut re-loads its im2col A panel for every
      // 128-column O chunk (ncu, layer2 block 0: 768 KB of L2->SM operand
      // traffic per 128-row tile, ~9 TB/s, the epilogue starved 25% of the time)
      if (!pl->chain_ds2 && C3.ds_op >= 0 && pl->layers[C3.ds_op].p[10] != 1) break;
      C3.chain_op = (int)j;
      C1.fused = true;
      break;
    }
  }
}

int upload_weights(b2_plan* pl, const uint8_t* data, const std::vector<WeightRec>& wr,
                   size_t data_len) {
  const bool bf = pl->dtype == B2_DT_BF16;
  auto wptr = [&](int idx, size_t* numel) -> const float* {
    if (idx < 0 || idx >= (int)wr.size()) return nullptr;
    if (wr[idx].offset + wr[idx].numel * 4 > data_len) return nullptr;
    *numel = wr[idx].numel;
    return reinterpret_cast<const float*>(data + wr[idx].offset);
  };
  for (Layer& L : pl->layers) {
    size_t n = 0, nb = 0;
    int rc = B2_OK;
    switch (L.kind) {
      case OP_CONV:
      case OP_LINEAR: {
        const bool conv = L.kind == OP_CONV;
        const int N = conv ? L.p[7] : L.p[5];
        const int K = conv ? L.p[8] * L.p[9] * L.p[6] : L.p[4];
        const float* w = wptr(L.p[2], &n);
        if (!w || n != (size_t)N * K) return fail(B2_ERR_FORMAT, "weight %d size mismatch", L.p[2]);
        if (L.ds_op >= 0) {
          // folded projection shortcut: one bias b3 + bd
          std::vector<float> bsum(N, 0.f);
          for (int src : {L.p[3], pl->layers[L.ds_op].p[3]}) {
            if (src < 0) continue;
            const float* bsrc = wptr(src, &nb);
            if (!bsrc || nb != (size_t)N) return fail(B2_ERR_FORMAT, "bias size mismatch");
            for (int j = 0; j < N; ++j) bsum[j] += bsrc[j];
          }
          if ((rc = upload_f32(pl, bsum.data(), bsum.size(), &L.bias))) return rc;
        } else if (L.p[3] >= 0) {
          const float* bsrc = wptr(L.p[3], &nb);
          if (!bsrc || nb != (size_t)N) return fail(B2_ERR_FORMAT, "bias size mismatch");
          if ((rc = upload_f32(pl, bsrc, nb, &L.bias))) return rc;
        }
        L.K = K;
        const bool plain = !conv || (L.p[8] == 1 && L.p[9] == 1 && L.p[10] == 1 && L.p[11] == 0);
        L.tc = bf && !pl->force_simt;
        if (L.tc) {
          const int C = conv ? L.p[6] : K;
          if (C % 8 != 0)
            return fail(B2_ERR_UNSUPPORTED, "bf16 %s needs channels %% 8 == 0 (got %d)",
                        conv ? "conv" : "linear", C);
          L.gather = !plain;
          const int R = conv ? L.p[8] : 1, S = conv ? L.p[9] : 1;
          const bool pow2 = (C & (C - 1)) == 0;
          L.gmode = !L.gather ? 0 : (C % 64 == 0) ? 1 : (S * C <= 64 && pow2) ? 2 : 3;
          if (L.gather && (L.gmode == 1 || (C == 8 && pl->im2col8)) && pl->use_im2col) {
            L.im2col = true;     // TMA im2col producer instead of the cp.async gather
            L.gather = false;
            L.im2col_mode = C == 8 ? 2 : 1;
            if (C == 8) L.gmode = 3;   // generic (r, s, c) K order, K padded to 64
            L.kpad = (K + 63) / 64 * 64;
            L.ldw = L.kpad;
          }
          L.kpad = L.gmode == 2 ? R * 64 : (K + 63) / 64 * 64;
          if (L.s2d) {
            L.gather = false;
            L.im2col = false;
            L.kpad = L.s2d_Rp * 64;
          }
          L.band8 = conv && pl->use_band && C == 8 && R == 3 && S == 3 && L.p[10] == 1 &&
                    L.p[11] == 1 && N % 64 == 0 && L.p[15] < 0 &&
                    (L.p[14] == ACT_NONE || L.p[14] == ACT_RELU) && L.p[12] == L.p[4] &&
                    L.p[13] == L.p[5] && !L.s2d;
          if (L.band8) {
            L.gather = false;
            L.im2col = false;
            L.kpad = 128;   // R * 32 = 96, padded to whole 64-wide weight blocks
          }
          L.ldw = L.kpad;
          std::vector<float> h((size_t)N * L.kpad, 0.f);
          if (L.band8) {
            for (int n = 0; n < N; ++n)
              for (int r = 0; r < 3; ++r)
                for (int ss = 0; ss < 3; ++ss)
                  for (int c = 0; c < 8; ++c)
                    h[(size_t)n * L.kpad + r * 32 + ss * 8 + c] =
                        w[(size_t)n * K + ((size_t)r * 3 + ss) * 8 + c];
          } else if (L.s2d) {
            // W''[n][r'][s'][q], q = (dy*2+dx)*4 + c  <-  W[n][2r'+dy-1][2s'+dx-1][c]
            for (int n = 0; n < N; ++n)
              for (int rp = 0; rp < L.s2d_Rp; ++rp)
                for (int sp = 0; sp < 4; ++sp)
                  for (int q = 0; q < 16; ++q) {
                    const int c = q & 3, dx = (q >> 2) & 1, dy = q >> 3;
                    const int r = 2 * rp + dy - 1, ss = 2 * sp + dx - 1;
                    if (c >= L.s2d_creal || r < 0 || r >= R || ss < 0 || ss >= S) continue;
                    h[(size_t)n * L.kpad + rp * 64 + sp * 16 + q] =
                        w[(size_t)n * K + ((size_t)r * S + ss) * C + c];
                  }
          } else if (L.gmode == 2) {   // [N][R][64]: each filter row's (s, c) run padded to 64
            for (int n = 0; n < N; ++n)
              for (int r = 0; r < R; ++r)
                memcpy(&h[(size_t)n * L.kpad + r * 64], w + (size_t)n * K + (size_t)r * S * C,
                       sizeof(float) * S * C);
          } else {
            for (int r = 0; r < N; ++r)
              memcpy(&h[(size_t)r * L.kpad], w + (size_t)r * K, sizeof(float) * K);
          }
          if ((rc = upload_as<bf16>(pl, h, &L.w))) return rc;
        } else if (!bf && !pl->force_simt && pl->use_tf32 &&
                   ((plain && (conv ? L.p[6] : L.p[9]) % 4 == 0 && K % 4 == 0) ||
                    (conv && L.p[6] % 32 == 0) || (conv && pl->tf32_gather))) {
          // 3xTF32: weights split once into hi (TF32-exact) and lo = w - hi,
          // [N][Kpad32] fp32
          L.tf32 = true;
          L.tf32_gather = conv && !plain && L.p[6] % 32 != 0;
          L.kpad = (K + 31) / 32 * 32;
          L.ldw = L.kpad;
          std::vector<float> hi((size_t)N * L.kpad, 0.f), lo((size_t)N * L.kpad, 0.f);
          for (int n = 0; n < N; ++n)
            for (int k = 0; k < K; ++k) {
              const float x = w[(size_t)n * K + k];
              uint32_t u;
              memcpy(&u, &x, 4);
              u &= 0xFFFFE000u;
              float xh;
              memcpy(&xh, &u, 4);
              hi[(size_t)n * L.kpad + k] = xh;
              lo[(size_t)n * L.kpad + k] = x - xh;
            }
          if ((rc = upload_as<float>(pl, hi, &L.w)) || (rc = upload_as<float>(pl, lo, &L.w2)))
            return rc;
        } else {
          L.ldw = K;
          std::vector<float> h(w, w + (size_t)N * K);
          if ((rc = bf ? upload_as<bf16>(pl, h, &L.w) : upload_as<float>(pl, h, &L.w)))
            return rc;
        }
        break;
      }
      case OP_DWCONV: {
        const int C = L.p[6], R = L.p[12];
        const float* w = wptr(L.p[2], &n);
        if (!w || n != (size_t)C * R * R) return fail(B2_ERR_FORMAT, "dw weight size mismatch");
        std::vector<float> h((size_t)C * R * R);
        for (int c = 0; c < C; ++c)
          for (int t = 0; t < R * R; ++t) h[(size_t)t * C + c] = w[(size_t)c * R * R + t];
        if ((rc = bf ? upload_as<bf16>(pl, h, &L.w) : upload_as<float>(pl, h, &L.w))) return rc;
        if (L.p[3] >= 0) {
          const float* bsrc = wptr(L.p[3], &nb);
          if (!bsrc || nb != (size_t)C) return fail(B2_ERR_FORMAT, "dw bias size mismatch");
          if ((rc = upload_f32(pl, bsrc, nb, &L.bias))) return rc;
        }
        break;
      }
      case OP_LAYERNORM: {
        const int D = L.p[4];
        const float* g = wptr(L.p[2], &n);
        const float* b = wptr(L.p[3], &nb);
        if (!g || !b || n != (size_t)D || nb != (size_t)D)
          return fail(B2_ERR_FORMAT, "layernorm params size mismatch");
        if ((rc = upload_f32(pl, g, n, &L.g))) return rc;
        if ((rc = upload_f32(pl, b, nb, &L.b))) return rc;
        break;
      }
      case OP_EMBED: {
        const int D = L.p[7], S = L.p[8], V = L.p[9];
        size_t n1, n2, n3, n4, n5;
        const float* word = wptr(L.p[2], &n1);
        const float* pos = wptr(L.p[3], &n2);
        const float* typ = wptr(L.p[4], &n3);
        const float* g = wptr(L.p[5], &n4);
        const float* b = wptr(L.p[6], &n5);
        if (!word || !pos || !typ || !g || !b || n1 != (size_t)V * D || n2 < (size_t)S * D ||
            n3 != (size_t)D || n4 != (size_t)D || n5 != (size_t)D)
          return fail(B2_ERR_FORMAT, "embedding tables size mismatch");
        std::vector<float> h1(word, word + n1), h2(pos, pos + (size_t)S * D), h3(typ, typ + n3);
        if (bf) {
          if ((rc = upload_as<bf16>(pl, h1, &L.w)) || (rc = upload_as<bf16>(pl, h2, &L.w2)) ||
              (rc = upload_as<bf16>(pl, h3, &L.w3)))
            return rc;
        } else {
          if ((rc = upload_as<float>(pl, h1, &L.w)) || (rc = upload_as<float>(pl, h2, &L.w2)) ||
              (rc = upload_as<float>(pl, h3, &L.w3)))
            return rc;
        }
        if ((rc = upload_f32(pl, g, n4, &L.g)) || (rc = upload_f32(pl, b, n5, &L.b))) return rc;
        break;
      }
      case OP_ATTENTION:
        L.tc = bf && !pl->force_simt && L.p[4] == 128 && L.p[3] == 64;
        break;
      default:
        break;
    }
  }
  return B2_OK;
}

size_t elem_size(const b2_plan* pl, int t) {
  if (pl->tensors[t].kind == 1) return 4;   // int32 ids
  return pl->dtype == B2_DT_BF16 ? 2 : 4;
}

int validate_ops(b2_plan* pl) {
  const int nt = (int)pl->tensors.size();
  auto tok = [&](int t) { return t >= 0 && t < nt; };
  for (size_t i = 0; i < pl->layers.size(); ++i) {
    const Layer& L = pl->layers[i];
    const int* p = L.p;
    bool ok = true;
    switch (L.kind) {
      case OP_INPUT: ok = tok(p[0]) && p[1] > 0 && p[4] >= p[1]; break;
      case OP_TOKENS:
        ok = tok(p[0]) && p[1] > 0 && p[2] > 0 && (!p[3] || tok(p[4])) &&
             pl->in_elems == (long)p[1] * (p[3] ? 2 : 1);
        pl->vocab = p[2];
        pl->seq = p[1];
        break;
      case OP_CONV: ok = tok(p[0]) && tok(p[1]) && (p[15] < 0 || tok(p[15])); break;
      case OP_LINEAR: ok = tok(p[0]) && tok(p[1]) && (p[8] < 0 || tok(p[8])); break;
      case OP_DWCONV: case OP_MAXPOOL: case OP_AVGPOOL: case OP_ACT: ok = tok(p[0]) && tok(p[1]); break;
      case OP_LAYERNORM: ok = tok(p[0]) && tok(p[1]) && (p[7] < 0 || tok(p[7])); break;
      case OP_EMBED: ok = tok(p[0]) && tok(p[1]); break;
      case OP_ATTENTION:
        ok = tok(p[0]) && tok(p[1]) && p[3] == 64 && (!p[5] || tok(p[6]));
        break;
      case OP_OUTPUT: {
        ok = p[0] >= 1 && p[0] <= 15;
        for (int j = 0; ok && j < p[0]; ++j)
          ok = tok(p[1 + 2 * j]) && p[2 + 2 * j] >= 0 &&
               p[2 + 2 * j] + (long)pl->tensors[p[1 + 2 * j]].elems <= pl->out_elems;
        break;
      }
      default: return fail(B2_ERR_UNSUPPORTED, "op %zu: unknown kind %d", i, L.kind);
    }
    if (!ok) return fail(B2_ERR_FORMAT, "op %zu (kind %d): bad parameters", i, L.kind);
  }
  return B2_OK;
}

// ------------------------------------------------------------------ forward
template <typename T>
int run_ops(b2_plan* pl, BatchState& S, const void* d_in, float* d_out, cudaStream_t st,
            cudaEvent_t* op_events) {
  const int B = S.batch;
  auto A = [&](int t) { return static_cast<T*>(S.act[t]); };
  int launches = 0;
  for (size_t li = 0; li < pl->layers.size(); ++li) {
    Layer& L = pl->layers[li];
    const int* p = L.p;
    if (op_events) {            // eager profile pass: one NVTX range per op
      if (li) nvtxRangePop();
      char nm[32];
      snprintf(nm, sizeof nm, "op %zu kind %d", li, L.kind);
      nvtxRangePushA(nm);
      CK(cudaEventRecord(op_events[li], st));
    }
    // fused 2-layer MLP: one launch at the input op, for batches <= 8 (measured:
    // b=1 22.4 -> 12.3 us; from b=16 on the four-launch path is faster, 22.5 vs
    // 33 us, the fused kernel's row-group tail being serial)
    if (pl->mlp_in >= 0 && S.mlp_ctr) {
      if ((int)li == pl->mlp_in) {
        const Layer &A = pl->layers[pl->mlp_l1], &Bl = pl->layers[pl->mlp_l2];
        MlpArgs m{};
        m.in = static_cast<const float*>(d_in);
        m.w1 = A.w;
        m.w1lo = A.tf32 ? A.w2 : nullptr;
        m.ldw1 = A.ldw;
        m.b1 = A.bias;
        m.act1 = A.p[7];
        m.w2 = Bl.w;
        m.w2lo = Bl.tf32 ? Bl.w2 : nullptr;
        m.ldw2 = Bl.ldw;
        m.b2 = Bl.bias;
        m.act2 = Bl.p[7];
        m.xin = S.act[p[0]];
        m.h = S.act[A.p[1]];
        m.y = S.act[Bl.p[1]];
        m.out = d_out;
        m.out_stride = (long)pl->out_elems;
        m.out_off = 0;
        m.B = B;
        m.K1 = A.p[4];
        m.N1 = A.p[5];
        m.N2 = Bl.p[5];
        m.counters = S.mlp_ctr;
        CK(mlp2<T>(m, st));
        ++launches;
        continue;
      }
      if ((int)li == pl->mlp_l1 || (int)li == pl->mlp_l2 || (int)li == pl->mlp_out) continue;
    }
    switch (L.kind) {
      case OP_INPUT:
        if (L.s2d)
          CK(input_pack_s2d(static_cast<const float*>(d_in), reinterpret_cast<bf16*>(S.act[p[0]]),
                            B, p[1], p[2], p[3], L.s2d_shift, L.s2d_H2, L.s2d_W2, st));
        else
          CK(input_pack<T>(static_cast<const float*>(d_in), A(p[0]), B, p[1], p[2], p[3], p[4],
                           st));
        ++launches;
        break;
      case OP_TOKENS:
        CK(tokens_pack(static_cast<const int64_t*>(d_in), static_cast<int32_t*>(S.act[p[0]]),
                       p[3] ? static_cast<uint32_t*>(S.act[p[4]]) : nullptr, B, p[1],
                       (int)pl->in_elems, p[2], st));
        ++launches;
        break;
      case OP_CONV:
      case OP_LINEAR: {
        if (L.fused) break;   // projection shortcut folded into the block's last conv
        const bool conv = L.kind == OP_CONV;
        const int N = conv ? p[7] : p[5];
        const long M = conv ? (long)B * p[12] * p[13] : (long)B * p[6];
        const int res_t = conv ? p[15] : p[8];
        const int act = conv ? p[14] : p[7];
        T* out = A(p[1]);
        if (L.tf32) {
          const bool plain = !conv || (p[8] == 1 && p[9] == 1 && p[10] == 1 && p[11] == 0);
          TcArgs a{};
          a.nsplit = 1;
          a.M = (int)M;
          a.N = N;
          a.kblocks = L.kpad / 32;
          a.bias = L.bias;
          a.res = res_t >= 0 ? reinterpret_cast<const bf16*>(S.act[res_t]) : nullptr;  // fp32 data
          a.ldres = N;
          a.out = reinterpret_cast<bf16*>(out);   // fp32 data
          a.ldo = N;
          a.act = act;
          a.tiles_m = (int)((M + 127) / 128);
          a.tiles_n = (N + 127) / 128;
          if (L.tf32_gather) {   // materialise the im2col rows, then a plain GEMM over them
            CK(im2col_f32(static_cast<const float*>(S.act[p[0]]), S.col, B, p[4], p[5], p[6], p[8],
                          p[9], p[10], p[11], p[12], p[13], L.kpad, st));
            ++launches;
          } else if (!plain) {
            a.a_im2col = 1;
            a.C = p[6];
            a.R = p[8];
            a.S = p[9];
            a.OW = p[13];
            a.OHW = p[12] * p[13];
            a.stride = p[10];
            a.pad = p[11];
          }
          CK(tf32_gemm_launch(a, S.tmA[li], S.tmB[li], S.tmI[li], pl->num_sms, st));
        } else if (L.tc && S.chain[li]) {
          ChainArgs ca = S.cargs[li];
          ca.reverse = pl->alt_order ? (launches & 1) : 0;
          CK(chain_launch(ca, S.tmA[li], S.tmB[li], S.tmR[li], S.tmI[li], S.tmB2[li], S.tmO[li],
                          S.tmT[li], pl->num_sms, st));
        } else if (L.tc && S.band[li] && L.pool_op >= 0) {
          CK(stem_pool_launch(S.bargs[li], S.tmA[li], S.tmB[li], pl->num_sms, st));
        } else if (L.tc && S.band[li]) {
          CK(conv_band_launch(S.bargs[li], S.bn[li], L.s2d ? 16 : L.band8 ? 8 : 64, S.tmA[li], S.tmB[li],
                              S.tmO[li], S.tmT[li], pl->num_sms, st));
        } else if (L.tc) {
          TcArgs a{};
          a.nsplit = 1;
          a.M = (int)M;
          a.N = N;
          a.kblocks = L.kpad / 64;
          a.Kreal = L.K;
          a.bias = L.bias;
          a.res = (res_t >= 0 && !S.fold[li]) ? reinterpret_cast<const bf16*>(S.act[res_t])
                                              : nullptr;
          a.ldres = N;
          a.out = reinterpret_cast<bf16*>(out);
          a.ldo = N;
          a.act = act;
          const int bn = S.bn[li];
          a.tiles_m = (int)((M + 127) / 128);
          if (L.s2d) {
            a.tiles_m = B * p[12];     // one output row per M tile
            a.OH = p[12];
            a.out3d = 1;
            a.a_im2col = 3;
          }
          a.tiles_n = (N + bn - 1) / bn;
          if (L.gather || L.im2col) {
            a.a_im2col = L.im2col ? L.im2col_mode : 0;
            a.R = p[8];
            a.x = reinterpret_cast<const bf16*>(S.act[p[0]]);
            a.H = p[4];
            a.W = p[5];
            a.C = p[6];
            a.OW = p[13];
            a.OHW = p[12] * p[13];
            a.S = p[9];
            a.stride = p[10];
            a.pad = p[11];
            a.gmode = L.gmode;
            int lg2 = 0;
            while ((1 << lg2) < p[6]) ++lg2;
            a.c_log2 = lg2;
            a.SC = p[9] * p[6];
          }
          a.tma_epi = bn >= 32 && N % 8 == 0 && pl->epi_mode != 2;
          a.a_narrow = S.a_narrow[li];
          a.epi_debug = pl->epi_mode == 2 ? 0 : pl->epi_mode;
          a.ts_debug = pl->ts_debug;
          a.stages = pl->stages_override;
          a.reverse = pl->alt_order ? (launches & 1) : 0;
          a.res_kblocks = S.fold[li] ? (bn >= 64 ? bn / 64 : 1) : 0;   // BN 32: one 64-wide block, identity rows [0, 32)
          if (S.fold[li] >= 2) {
            const int* q = pl->layers[L.ds_op].p;
            a.res_kblocks = pl->layers[L.ds_op].kpad / 64;
            a.fold_kind = S.fold[li] - 1;   // 1: stride-1 shortcut, 2: strided (im2col)
            a.ds_H = q[4];
            a.ds_W = q[5];
            a.OW = q[13];
            a.OHW = q[12] * q[13];
            a.stride = q[10];
          }
          if (S.pair[li]) {
            a.tiles_m = (int)((M + 255) / 256);
            CK(tc_gemm2_launch(a, bn, S.tmA[li], S.tmB[li], S.tmO[li],
                               S.fold[li] ? S.tmR[li] : S.tmO[li],
                               S.fold[li] ? S.tmI[li] : S.tmO[li], pl->num_sms, st));
          } else if (S.split[li] > 1) {
            a.nsplit = S.split[li];
            a.ws = S.ws;
            a.res = nullptr;
            a.res_kblocks = 0;
            CK(tc_gemm_launch(a, bn, false, S.tmA[li], S.tmB[li], S.tmO[li], S.tmO[li], S.tmO[li],
                              pl->num_sms, st));
            CK(splitk_finalize(S.ws, a.nsplit, L.bias,
                               res_t >= 0 ? reinterpret_cast<const bf16*>(S.act[res_t]) : nullptr,
                               reinterpret_cast<bf16*>(out), M, N, act, st));
            ++launches;
          } else {
            CK(tc_gemm_launch(a, bn, L.gather, L.gather ? S.tmB[li] : S.tmA[li], S.tmB[li],
                              S.tmO[li], S.fold[li] ? S.tmR[li] : S.tmO[li],
                              S.fold[li] ? S.tmI[li] : S.tmO[li], pl->num_sms, st));
          }
        } else {
          GemmSimtArgs a{};
          a.M = (int)M;
          a.N = N;
          a.K = L.K;
          a.a = S.act[p[0]];
          a.lda = conv ? L.K : p[9];
          a.w = L.w;
          a.ldw = L.ldw;
          a.bias = L.bias;
          a.res = res_t >= 0 ? S.act[res_t] : nullptr;
          a.out = out;
          a.act = act;
          a.conv = conv && !(p[8] == 1 && p[9] == 1 && p[10] == 1 && p[11] == 0);
          if (conv) {
            if (!a.conv) a.lda = p[6];
            a.H = p[4];
            a.W = p[5];
            a.C = p[6];
            a.OW = p[13];
            a.OHW = p[12] * p[13];
            a.S = p[9];
            a.stride = p[10];
            a.pad = p[11];
          }
          CK(gemm_simt<T>(a, st));
        }
        ++launches;
        break;
      }
      case OP_DWCONV:
        CK(dwconv<T>(A(p[0]), static_cast<const T*>(L.w), L.bias, A(p[1]), B, p[4], p[5], p[6],
                     p[12], p[7], p[8], p[9], p[10], p[11], st));
        ++launches;
        break;
      case OP_MAXPOOL:
        if (L.fused) break;   // computed by the producing stem's epilogue
        CK(maxpool<T>(A(p[0]), A(p[1]), B, p[2], p[3], p[4], p[5], p[6], p[7], p[8], p[9], st));
        ++launches;
        break;
      case OP_AVGPOOL:
        CK(avgpool<T>(A(p[0]), A(p[1]), B, p[2] * p[3], p[4], st));
        ++launches;
        break;
      case OP_LAYERNORM: {
        float eps;
        memcpy(&eps, &p[6], 4);
        CK(layernorm<T>(A(p[0]), p[7] >= 0 ? A(p[7]) : nullptr, L.g, L.b, A(p[1]),
                        (long)B * p[5], p[4], eps, st));
        ++launches;
        break;
      }
      case OP_EMBED: {
        float eps;
        memcpy(&eps, &p[10], 4);
        CK(embed_ln<T>(static_cast<const int32_t*>(S.act[p[0]]), static_cast<const T*>(L.w),
                       static_cast<const T*>(L.w2), static_cast<const T*>(L.w3), L.g, L.b,
                       A(p[1]), B, p[8], p[7], eps, st));
        ++launches;
        break;
      }
      case OP_ATTENTION:
      {
        const uint32_t* km = p[5] ? static_cast<const uint32_t*>(S.act[p[6]]) : nullptr;
        if (L.tc)
          CK(attention_tc(S.tmA[li], reinterpret_cast<bf16*>(S.act[p[1]]), B, p[2], km, st));
        else
          CK(attention<T>(A(p[0]), A(p[1]), B, p[4], p[2], p[3], km, st));
      }
        ++launches;
        break;
      case OP_ACT:
        CK(act_ew<T>(A(p[0]), A(p[1]), (long)B * p[2], p[3], st));
        ++launches;
        break;
      case OP_OUTPUT:
        for (int j = 0; j < p[0]; ++j) {
          const int t = p[1 + 2 * j];
          CK(output_gather<T>(A(t), d_out, B, pl->tensors[t].elems, pl->out_elems, p[2 + 2 * j],
                              st));
          ++launches;
        }
        break;
    }
  }
  if (op_events && !pl->layers.empty()) nvtxRangePop();
  pl->launches = launches;
  return B2_OK;
}

int run_forward(b2_plan* pl, BatchState& S, const void* d_in, float* d_out, cudaStream_t st,
                cudaEvent_t* ev = nullptr) {
  return pl->dtype == B2_DT_BF16 ? run_ops<bf16>(pl, S, d_in, d_out, st, ev)
                                 : run_ops<float>(pl, S, d_in, d_out, st, ev);
}

size_t in_bytes(const b2_plan* pl, int batch) {
  return (size_t)batch * pl->in_elems * (pl->input_kind == B2_IN_TOKENS_I64 ? 8 : 4);
}

// Tensor maps and arguments of a chained block tail (plan_chain).  Returns 1
// when set up, -code on error.
int plan_chain_state(b2_plan* pl, BatchState& S, size_t li, int batch) {
  Layer& L = pl->layers[li];
  if (L.chain_op < 0) return 0;
  const int* p = L.p;
  const Layer& C1 = pl->layers[L.chain_op];
  const int N1 = p[7], N2 = C1.p[7];
  const long M = (long)batch * p[12] * p[13];
  ChainArgs a{};
  a.M = (int)M;
  a.N1 = N1;
  a.N2 = N2;
  a.kblocks = L.kpad / 64;
  a.tiles_m = (int)((M + 127) / 128);
  a.bias1 = L.bias ? L.bias : pl->zero_bias;
  a.bias2 = C1.bias ? C1.bias : pl->zero_bias;
  bool ok = make_tmap_bf16(&S.tmA[li], S.act[p[0]], (uint64_t)M, (uint64_t)L.K,
                           (uint64_t)p[6] * 2, 128) &&
            make_tmap_bf16(&S.tmB[li], L.w, (uint64_t)N1, (uint64_t)L.kpad, (uint64_t)L.kpad * 2,
                           128) &&
            make_tmap_bf16(&S.tmB2[li], C1.w, (uint64_t)N2, (uint64_t)C1.kpad,
                           (uint64_t)C1.kpad * 2, (uint32_t)N2) &&
            make_tmap_bf16(&S.tmO[li], S.act[p[1]], (uint64_t)M, (uint64_t)N1, (uint64_t)N1 * 2,
                           128) &&
            make_tmap_bf16(&S.tmT[li], S.act[C1.p[1]], (uint64_t)M, (uint64_t)N2,
                           (uint64_t)N2 * 2, 128);
  if (L.ds_op >= 0) {
    const Layer& D = pl->layers[L.ds_op];
    const int* q = D.p;
    if (q[10] == 1)
      ok = ok && make_tmap_bf16(&S.tmR[li], S.act[q[0]], (uint64_t)M, (uint64_t)q[6],
                                (uint64_t)q[6] * 2, 128);
    else
      ok = ok && make_tmap_im2col(&S.tmR[li], S.act[q[0]], batch, q[4], q[5], q[6], 1, 1, q[10],
                                  0, 64);
    ok = ok && make_tmap_bf16(&S.tmI[li], D.w, (uint64_t)N1, (uint64_t)D.kpad,
                              (uint64_t)D.kpad * 2, 128);
    a.res_kblocks = D.kpad / 64;
    a.fold_kind = q[10] == 1 ? 1 : 2;
    a.OW = q[13];
    a.OHW = q[12] * q[13];
    a.stride = q[10];
  } else {
    ok = ok && make_tmap_bf16(&S.tmR[li], S.act[p[15]], (uint64_t)M, (uint64_t)N1,
                              (uint64_t)N1 * 2, 128) &&
         make_tmap_bf16(&S.tmI[li], pl->identity, 256, 256, 512, 128);
    a.res_kblocks = 2;             // 128 residual columns per O chunk
    a.fold_kind = 0;
  }
  if (!ok) return -fail(B2_ERR_CUDA, "layer %zu: chain tensor maps rejected", li);
  if (!chain_config(a)) return -fail(B2_ERR_UNSUPPORTED, "layer %zu: chain does not fit", li);
  S.chain[li] = 1;
  S.cargs[li] = a;
  return 1;
}

// Banded implicit-GEMM conv (conv_band.cu) for stride-1 "same" k x k convs
// with C % 64 == 0 and for space-to-depth stems.  Returns 1 when layer li
// runs banded (tensor maps built), 0 to keep the gemm_tc path, -code on error.
// Band row pitch: padded width rounded so 32-position epilogue chunks never
// straddle an output row at a nonzero column (multiple of 32, or 8 / 16).
int band_pitch(int w) { return w <= 8 ? 8 : w <= 16 ? 16 : (w + 31) / 32 * 32; }

int plan_band(b2_plan* pl, BatchState& S, size_t li, int batch) {
  Layer& L = pl->layers[li];
  const int* p = L.p;
  if ((!pl->use_band && !L.band8) || L.kind != OP_CONV || p[15] >= 0) return 0;
  const int C = p[6], N = p[7], R = p[8], Sf = p[9], stride = p[10], pad = p[11];
  const int OH = p[12], OW = p[13];
  BandArgs a{};
  int cgw = 64;
  if (L.s2d) {
    // N = 32 (MobileNetV2 stem) runs as a 64-wide tile: weight rows 32..63 are
    // TMA zero-fill and the output map clips columns >= 32
    if ((N % 64 != 0 && N != 32) || N > 128) return 0;
    cgw = 16;
    a.Wp = band_pitch(L.s2d_W2);
    a.R = L.s2d_Rp;
    a.S = 4;   // the s2d weight layout always holds 4 columns of 16 (zeros past the filter)
    a.CG = 1;
    a.x0 = a.y0 = 0;
  } else if (L.band8) {
    cgw = 8;
    a.Wp = band_pitch(OW + 2);
    a.R = a.S = 3;
    a.CG = 1;
    a.x0 = a.y0 = -1;
  } else {
    // N >= 256: the im2col GEMM's wide tiles already amortise A (measured:
    // band 62.8 / 108 us vs im2col 60.8 / 99.7 us on ResNet layer3 / layer4)
    if (N > pl->band_max_n) return 0;
    if (!L.im2col || stride != 1 || R != Sf || (R & 1) == 0 || pad != (R - 1) / 2 ||
        OH != p[4] || OW != p[5] || C % 64 != 0 || N % 64 != 0 || R == 1)
      return 0;
    a.Wp = band_pitch(OW + Sf - 1);
    a.R = R;
    a.S = Sf;
    a.CG = C / 64;
    a.x0 = a.y0 = -pad;
    a.pool2 = L.pool2_op >= 0 ? 1 : 0;   // band_config: even band heights, streamed weights
  }
  const int bn = N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : 64;
  if (cgw == 16 && bn > 128) return 0;
  a.B = batch;
  a.H = OH;
  a.W = OW;
  a.N = N;
  a.kblocks = L.kpad / 64;
  a.tiles_n = (N + bn - 1) / bn;
  a.out = reinterpret_cast<bf16*>(S.act[p[1]]);
  a.act = p[14];
  a.bias = L.bias ? L.bias : pl->zero_bias;
  a.nseg = 1;
  a.seg_w = OW;
  if (L.pool_op >= 0) {
    const int* q = pl->layers[L.pool_op].p;
    a.pout = reinterpret_cast<bf16*>(S.act[q[1]]);
    a.PH = q[8];
    a.PW = q[9];
    if (!stem_pool_config(a))
      return -fail(B2_ERR_UNSUPPORTED, "layer %zu: fused stem/max-pool geometry rejected", li);
  } else if ((L.pool2_op >= 0 && a.Wp > 128) || !band_config(a, bn, cgw) ||
             !band_supported(a, bn, cgw, a.act)) {
    // rows too wide for one band pitch (VGG 224x224): split each row into two
    // column segments of pitch 128 (126 valid columns + halo).  The fused
    // 2x2 pool needs exactly one output row per M tile, so it always splits.
    if (L.s2d || a.Wp <= 128 || OW > 2 * (128 - (Sf - 1))) return 0;
    a.Wp = 128;
    a.seg_w = 128 - (Sf - 1);
    a.nseg = (OW + a.seg_w - 1) / a.seg_w;
    if (!band_config(a, bn, cgw) || !band_supported(a, bn, cgw, a.act)) return 0;
  }
  if (L.pool_op < 0 && L.pool2_op < 0 &&
      (long)a.B * a.nbands * a.tiles_n < pl->num_sms) {   // small batch: more, smaller units
    BandArgs t = a;
    if (band_config(t, bn, cgw, 1) && band_supported(t, bn, cgw, t.act)) a = t;
  }
  // CTA pair (M = 256 UMMAs over two bands): N = 64 with resident weights,
  // when there are enough bands to give every pair of SMs work.  Measured:
  // ResNet layer1 3x3 b=256 69 -> 66 us; VGG 224x224 (two column segments per
  // row) 1.05 -> 1.34 ms, so single-segment rows only
  if (pl->band_pair && cgw == 64 && bn == 64 && a.CG == 1 && a.b_resident && a.tiles_n == 1 &&
      a.R == 3 && a.S == 3 && L.pool_op < 0 && L.pool2_op < 0 && a.nseg == 1 &&
      (long)a.B * a.nbands * a.nseg >= pl->num_sms) {
    BandArgs t = a;
    t.pair = 1;
    if (band_smem_bytes(t, 64) <= 232448) a = t;
  }
  if (L.pool2_op >= 0) {
    // the pool is already marked fused: this layer must take the pooling band path
    if (a.Wp != 128 || (a.bh > 1 && (a.bh & 1)) || (a.bh == 1 && (a.nbands & 1)) || a.R != 3 ||
        a.act != ACT_RELU ||
        !((bn == 64 && a.b_resident && a.CG == 1 && a.bh == 1) || (bn == 128 && !a.b_resident)))
      return -fail(B2_ERR_UNSUPPORTED,
                   "layer %zu: fused 2x2 max-pool band geometry rejected (Wp %d bh %d bn %d "
                   "resident %d CG %d act %d)", li, a.Wp, a.bh, bn, a.b_resident, a.CG, a.act);
    a.pool2 = 1;
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return -fail(B2_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int cin = L.s2d ? 16 : C;
  const int win = L.s2d ? L.s2d_W2 : p[5];
  const int hin = L.s2d ? L.s2d_H2 : p[4];
  cuuint64_t dims[4] = {(cuuint64_t)cin, (cuuint64_t)win, (cuuint64_t)hin, (cuuint64_t)batch};
  cuuint64_t str[3] = {(cuuint64_t)cin * 2, (cuuint64_t)win * cin * 2,
                       (cuuint64_t)hin * win * cin * 2};
  const int box_h = L.pool_op >= 0 ? 3 + a.R - 1 : a.bh + a.R - 1;
  cuuint32_t box[4] = {(cuuint32_t)cgw, (cuuint32_t)a.Wp, (cuuint32_t)box_h, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (fn(&S.tmA[li], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, S.act[p[0]], dims, str, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE,
         cgw == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                   : cgw == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -fail(B2_ERR_CUDA, "layer %zu: band A tensor map rejected", li);
  if (!make_tmap_bf16(&S.tmB[li], L.w, (uint64_t)N, (uint64_t)L.kpad, (uint64_t)L.kpad * 2,
                      (uint32_t)(a.pair ? bn / 2 : bn)))
    return -fail(B2_ERR_CUDA, "layer %zu: band B tensor map rejected", li);
  // output NHWC [B, OH, OW, N]: 32-channel x 32-pixel boxes, 64 B swizzle;
  // one map per column segment, each clipping at its own width
  // fused 2x2 pool: the maps describe the pooled tensor [B, OH/2, OW/2, N]
  // (16-pixel boxes), segment column offsets halved
  const int dv = a.pool2 ? 2 : 1;
  void* obase = a.pool2 ? S.act[pl->layers[L.pool2_op].p[1]] : S.act[p[1]];
  for (int sg = 0; sg < a.nseg && sg < 2; ++sg) {
    const int w0 = sg * a.seg_w, wn = sg + 1 < a.nseg ? a.seg_w : OW - w0;
    cuuint64_t odims[4] = {(cuuint64_t)N, (cuuint64_t)(wn / dv), (cuuint64_t)(OH / dv),
                           (cuuint64_t)batch};
    cuuint64_t ostr[3] = {(cuuint64_t)N * 2, (cuuint64_t)(OW / dv) * N * 2,
                          (cuuint64_t)(OH / dv) * (OW / dv) * N * 2};
    cuuint32_t obox[4] = {32, (cuuint32_t)(32 / dv), 1, 1};
    CUtensorMap* m = sg == 0 ? &S.tmO[li] : &S.tmT[li];
    if (fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, static_cast<bf16*>(obase) + (size_t)(w0 / dv) * N,
           odims, ostr, obox, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -fail(B2_ERR_CUDA, "layer %zu: band output tensor map rejected", li);
  }
  if (a.nseg > 2) return -fail(B2_ERR_UNSUPPORTED, "layer %zu: > 2 band segments", li);
  if (a.nseg == 1) S.tmT[li] = S.tmO[li];
  S.bn[li] = bn;
  S.band[li] = 1;
  S.bargs[li] = a;
  return 1;
}

int get_state(b2_plan* pl, int batch, BatchState** out) {
  auto it = pl->states.find(batch);
  if (it != pl->states.end()) {
    *out = &it->second;
    return B2_OK;
  }
  BatchState S;
  S.batch = batch;
  S.act.resize(pl->tensors.size(), nullptr);
  // one arena per batch size (one cudaMalloc + one memset instead of one per
  // tensor: ~0.3 s of first-cell set-up at ResNet b=256); 1 KB-aligned slices
  std::vector<size_t> off(pl->tensors.size());
  size_t arena = 0;
  for (size_t t = 0; t < pl->tensors.size(); ++t) {
    size_t bytes = (size_t)batch * pl->tensors[t].elems * elem_size(pl, (int)t);
    for (const Layer& L : pl->layers)   // space-to-depth input: [B, H2, W2, 16] bf16
      if (L.kind == OP_INPUT && L.s2d && L.p[0] == (int)t)
        bytes = (size_t)batch * L.s2d_H2 * L.s2d_W2 * 16 * 2;
    off[t] = arena;
    arena += (bytes + 256 + 1023) / 1024 * 1024;
  }
  CK(dmalloc(pl, (void**)&S.arena, arena));
  CK(cudaMemset(S.arena, 0, arena));
  for (size_t t = 0; t < pl->tensors.size(); ++t) S.act[t] = static_cast<uint8_t*>(S.arena) + off[t];
  CK(dmalloc(pl, (void**)&S.d_in, in_bytes(pl, batch) + 256));
  CK(cudaMemset(S.d_in, 0, in_bytes(pl, batch) + 256));
  if (pl->mlp_in >= 0 && batch <= 8) {
    const size_t groups = (size_t)(batch + 15) / 16;
    CK(dmalloc(pl, (void**)&S.mlp_ctr, groups * sizeof(unsigned) + 256));
    CK(cudaMemset(S.mlp_ctr, 0, groups * sizeof(unsigned) + 256));
  }
  CK(dmalloc(pl, (void**)&S.d_out, (size_t)batch * pl->out_elems * 4 + 256));
  S.bn.assign(pl->layers.size(), 0);
  S.tmA.resize(pl->layers.size());
  S.tmB.resize(pl->layers.size());
  S.tmO.resize(pl->layers.size());
  S.tmR.resize(pl->layers.size());
  S.fold.assign(pl->layers.size(), 0);
  S.a_narrow.assign(pl->layers.size(), 0);
  S.tmI.resize(pl->layers.size());
  S.band.assign(pl->layers.size(), 0);
  S.pair.assign(pl->layers.size(), 0);
  S.chain.assign(pl->layers.size(), 0);
  S.split.assign(pl->layers.size(), 1);
  size_t ws_elems = 0;
  size_t col_elems = 0;
  S.cargs.resize(pl->layers.size());
  S.tmB2.resize(pl->layers.size());
  S.tmT.resize(pl->layers.size());
  S.bargs.resize(pl->layers.size());
  for (size_t li = 0; li < pl->layers.size(); ++li) {
    Layer& L = pl->layers[li];
    if (L.tf32) {
      const int* p = L.p;
      const bool conv = L.kind == OP_CONV;
      const int N = conv ? p[7] : p[5];
      const long M = conv ? (long)batch * p[12] * p[13] : (long)batch * p[6];
      const bool plain = !conv || (p[8] == 1 && p[9] == 1 && p[10] == 1 && p[11] == 0);
      bool ok;
      if (L.tf32_gather) {   // A = the materialised im2col rows
        col_elems = std::max(col_elems, (size_t)M * L.kpad);
        continue;            // map made once `col` exists (below)
      }
      if (plain) {
        const long ld = conv ? p[6] : p[9];
        ok = make_tmap_f32(&S.tmA[li], S.act[p[0]], (uint64_t)M, (uint64_t)L.K,
                           (uint64_t)ld * 4, 128);
      } else {
        ok = make_tmap_im2col(&S.tmA[li], S.act[p[0]], batch, p[4], p[5], p[6], p[8], p[9],
                              p[10], p[11], 32, 4);
      }
      ok = ok && make_tmap_f32(&S.tmB[li], L.w, (uint64_t)N, (uint64_t)L.kpad,
                               (uint64_t)L.kpad * 4, 128) &&
           make_tmap_f32(&S.tmI[li], L.w2, (uint64_t)N, (uint64_t)L.kpad, (uint64_t)L.kpad * 4,
                         128);
      if (!ok) return fail(B2_ERR_CUDA, "layer %zu: 3xTF32 tensor maps rejected", li);
      continue;
    }
    if (!L.tc) continue;
    const int* p = L.p;
    int brc = plan_band(pl, S, li, batch);
    if (brc < 0) return -brc;
    if (brc == 1) continue;
    if (L.band8)   // its weights are in the paired-tap layout only conv_band reads
      return fail(B2_ERR_UNSUPPORTED, "layer %zu: 8-channel band conv geometry rejected", li);
    if (L.pool2_op >= 0)   // its max-pool was fused away at plan creation
      return fail(B2_ERR_UNSUPPORTED, "layer %zu: fused 2x2 max-pool needs the band kernel", li);
    brc = plan_chain_state(pl, S, li, batch);
    if (brc < 0) return -brc;
    if (brc == 1) continue;
    if (L.kind == OP_ATTENTION) {
      const uint64_t cols = 3ull * p[2] * p[3];
      if (!make_tmap_bf16(&S.tmA[li], S.act[p[0]], (uint64_t)batch * p[4], cols, cols * 2, 128))
        return fail(B2_ERR_CUDA, "layer %zu: cuTensorMapEncodeTiled(qkv) failed", li);
      continue;
    }
    const bool conv = L.kind == OP_CONV;
    const int N = conv ? p[7] : p[5];
    const long M = conv ? (long)batch * p[12] * p[13] : (long)batch * p[6];
    // CTA-pair (cta_group::2) GEMM vs single CTA and the tile width: per-SM
    // clock model in tc_pick_config (TMA fill rate vs MMA vs epilogue writes).
    // Pairs need a TMA-fed A (no gather / s2d / folded shortcut).
    const bool pair_allowed = pl->use_pair && !L.s2d && !L.gather &&
                              (!L.im2col || L.im2col_mode == 1) && N % 8 == 0 &&
                              M >= pl->pair_min_m && L.K >= pl->pair_min_k;
    const int res_in = conv ? p[15] : p[8];
    const int ds_kb = L.ds_op >= 0 ? pl->layers[L.ds_op].kpad / 64 : 0;   // folded shortcut K
    bool pair_ok = false;
    int bn = tc_pick_config(M, N, L.kpad / 64 + ds_kb, res_in >= 0 && L.K <= pl->fold_max_k,
                            pl->num_sms, pair_allowed, &pair_ok);
    // Memory-bound shapes (one K block, or im2col A that each extra N tile
    // re-gathers) want the widest tile: measured 56x56x64->256 128 -> 115 us,
    // 56x56x256->28x28x512/s2 110 -> 72 us with BN = 256 instead of 128.
    if (!pair_ok && N % 256 == 0 && (L.kpad <= 64 || (L.im2col && L.im2col_mode == 1))) bn = 256;
    if (pl->force_bn && !pair_ok && N % pl->force_bn == 0) bn = pl->force_bn;   // B2_FORCE_BN (tuning aid)
    S.bn[li] = bn;
    S.pair[li] = pair_ok;
    if (pl->verbose)
      fprintf(stderr, "b2: layer %zu M=%ld N=%d K=%d kpad=%d -> bn=%d pair=%d\n", li, M, N, L.K,
              L.kpad, bn, (int)pair_ok);
    if (!pair_ok && !L.gather && !L.s2d && L.ds_op < 0 && bn >= 32 && N % 8 == 0 &&
        pl->use_split && pl->epi_mode == 0) {
      const long tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
      const int sp = tc_pick_split(tiles, L.kpad / 64, pl->num_sms);
      if (sp > 1) {
        S.split[li] = sp;
        ws_elems = std::max(ws_elems, (size_t)sp * M * N);
      }
    }
    const uint32_t bbox = pair_ok ? bn / 2 : bn;
    if (!make_tmap_bf16(&S.tmB[li], L.w, (uint64_t)N, (uint64_t)L.kpad, (uint64_t)L.kpad * 2,
                        bbox))
      return fail(B2_ERR_CUDA, "layer %zu: cuTensorMapEncodeTiled(B) failed", li);
    if (L.s2d) {
      // A: overlapping 4D view of the space-to-depth input — element (k, ow, Y, n)
      // at ((n*H2 + Y)*W2 + ow)*16 + k: one 128 B row = 4 pixel columns x 16 ch
      EncodeTiledFn fn = encode_fn();
      cuuint64_t dims[4] = {64, (cuuint64_t)p[13], (cuuint64_t)L.s2d_H2, (cuuint64_t)batch};
      cuuint64_t str[3] = {32, (cuuint64_t)L.s2d_W2 * 32, (cuuint64_t)L.s2d_H2 * L.s2d_W2 * 32};
      cuuint32_t box[4] = {64, 128, 1, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      // out: [B*OH, OW, N] so the 32-row store boxes clip at the row end
      cuuint64_t odims[3] = {(cuuint64_t)N, (cuuint64_t)p[13], (cuuint64_t)batch * p[12]};
      cuuint64_t ostr[2] = {(cuuint64_t)N * 2, (cuuint64_t)N * p[13] * 2};
      cuuint32_t obox[3] = {32, 32, 1};
      cuuint32_t oes[3] = {1, 1, 1};
      if (!fn || N % 8 != 0 || bn < 32 ||
          fn(&S.tmA[li], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, S.act[p[0]], dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
          fn(&S.tmO[li], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, S.act[p[1]], odims, ostr, obox, oes,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(B2_ERR_CUDA, "layer %zu: space-to-depth tensor maps rejected", li);
      continue;
    }
    if (bn >= 32 && N % 8 == 0) {
      if (!make_tmap_bf16(&S.tmO[li], S.act[p[1]], (uint64_t)M, (uint64_t)N, (uint64_t)N * 2, 32,
                          32, CU_TENSOR_MAP_SWIZZLE_64B))
        return fail(B2_ERR_CUDA, "layer %zu: cuTensorMapEncodeTiled(out) failed", li);
    }
    // residual fold: cheap in MMA time when K is small, and it moves the
    // residual read out of the epilogue into the TMA pipeline
    const int res_t = conv ? p[15] : p[8];
    if (L.ds_op >= 0) {
      // folded shortcut: A = its input x (2D for stride 1, im2col for stride 2),
      // B = its weights; K blocks appended after this conv's own
      const Layer& D = pl->layers[L.ds_op];
      const int* q = D.p;
      bool ok;
      if (q[10] == 1)
        ok = make_tmap_bf16(&S.tmR[li], S.act[q[0]], (uint64_t)M, (uint64_t)q[6],
                            (uint64_t)q[6] * 2, 128);
      else
        ok = make_tmap_im2col(&S.tmR[li], S.act[q[0]], batch, q[4], q[5], q[6], 1, 1, q[10], 0, 64);
      if (!ok || !make_tmap_bf16(&S.tmI[li], D.w, (uint64_t)N, (uint64_t)D.kpad,
                                 (uint64_t)D.kpad * 2, bbox))
        return fail(B2_ERR_CUDA, "layer %zu: folded shortcut tensor maps rejected", li);
      S.fold[li] = q[10] == 1 ? 2 : 3;
    } else if (res_t >= 0 && bn >= 32 && N % 8 == 0 && L.K <= pl->fold_max_k && pl->identity &&
               S.split[li] == 1) {   // split-K adds the residual in its finalize pass
      if (!make_tmap_bf16(&S.tmR[li], S.act[res_t], (uint64_t)M, (uint64_t)N, (uint64_t)N * 2,
                          128) ||
          !make_tmap_bf16(&S.tmI[li], pl->identity, 256, 256, 512, bbox))
        return fail(B2_ERR_CUDA, "layer %zu: cuTensorMapEncodeTiled(res/identity) failed", li);
      S.fold[li] = 1;
    }
    if (L.im2col) {
      if (!make_tmap_im2col(&S.tmA[li], S.act[p[0]], batch, p[4], p[5], p[6], p[8], p[9], p[10],
                            p[11], L.im2col_mode == 2 ? 8 : 64))
        return fail(B2_ERR_CUDA, "layer %zu: cuTensorMapEncodeIm2col failed", li);
    } else if (!L.gather) {
      const int K = L.K;
      const long ld = conv ? p[6] : p[9];
      if ((ld * 2) % 16 != 0) return fail(B2_ERR_UNSUPPORTED, "layer %zu: A pitch not 16B", li);
      // K <= 32 on the single-CTA kernel: a 32- or 16-wide A box (64 B / 32 B
      // swizzle) instead of a half-empty 64-wide one — measured, boxes with
      // out-of-bounds halves stream at ~60% of the in-bounds rate
      const int nar = (pl->narrow_k && !S.pair[li] && S.split[li] == 1 && K <= 32)
                          ? (K <= 16 ? 16 : 32) : 0;
      S.a_narrow[li] = (char)nar;
      if (!make_tmap_bf16(&S.tmA[li], S.act[p[0]], (uint64_t)M, (uint64_t)K, (uint64_t)ld * 2, 128,
                          nar ? nar : 64,
                          nar == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                    : nar == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_128B))
        return fail(B2_ERR_CUDA, "layer %zu: cuTensorMapEncodeTiled(A) failed", li);
    }
  }
  if (col_elems) {
    CK(dmalloc(pl, (void**)&S.col, col_elems * sizeof(float) + 256));
    for (size_t li = 0; li < pl->layers.size(); ++li) {
      const Layer& L = pl->layers[li];
      if (!L.tf32_gather) continue;
      const int* p = L.p;
      const int N = p[7];
      const long M = (long)batch * p[12] * p[13];
      if (!make_tmap_f32(&S.tmA[li], S.col, (uint64_t)M, (uint64_t)L.kpad, (uint64_t)L.kpad * 4,
                         128) ||
          !make_tmap_f32(&S.tmB[li], L.w, (uint64_t)N, (uint64_t)L.kpad, (uint64_t)L.kpad * 4,
                         128) ||
          !make_tmap_f32(&S.tmI[li], L.w2, (uint64_t)N, (uint64_t)L.kpad, (uint64_t)L.kpad * 4,
                         128))
        return fail(B2_ERR_CUDA, "layer %zu: gathered 3xTF32 tensor maps rejected", li);
    }
  }
  if (ws_elems) {
    CK(dmalloc(pl, (void**)&S.ws, ws_elems * sizeof(float) + 256));
    CK(cudaMemset(S.ws, 0, ws_elems * sizeof(float) + 256));
  }
  // The memsets above run on the legacy default stream, which does not order
  // against the plan's non-blocking stream: without this the first forward at
  // a new batch size raced the zeroing of its own activation arena (seen as
  // wrong early rows on the first predict at b=256, right on the second).
  CK(cudaDeviceSynchronize());
  auto res = pl->states.emplace(batch, std::move(S));
  *out = &res.first->second;
  return B2_OK;
}

int enqueue(b2_plan* pl, BatchState& S, const void* d_in, float* d_out, cudaStream_t st) {
  return run_forward(pl, S, d_in, d_out, st);
}

// graph of the whole forward on the state's internal buffers (second = the
// alternate input/output pair used by the pipelined e2e loop)
int graph_of(b2_plan* pl, BatchState& S, cudaGraphExec_t* out, bool second = false) {
  cudaGraphExec_t& slot = second ? S.graph2 : S.graph;
  if (slot) {
    *out = slot;
    return B2_OK;
  }
  if (second && !S.d_in2) {
    CK(dmalloc(pl, (void**)&S.d_in2, in_bytes(pl, S.batch) + 256));
    CK(cudaMemset(S.d_in2, 0, in_bytes(pl, S.batch) + 256));
    CK(dmalloc(pl, (void**)&S.d_out2, (size_t)S.batch * pl->out_elems * 4 + 256));
    CK(cudaDeviceSynchronize());   // legacy-stream memset vs the plan's non-blocking stream
  }
  int rc;
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(pl->stream, cudaStreamCaptureModeThreadLocal));
  rc = run_forward(pl, S, second ? S.d_in2 : S.d_in, second ? S.d_out2 : S.d_out, pl->stream);
  cudaError_t e = cudaStreamEndCapture(pl->stream, &g);
  if (rc) return rc;
  if (e != cudaSuccess) return fail(B2_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
  CK(cudaGraphInstantiate(&slot, g, 0));
  cudaGraphDestroy(g);
  *out = slot;
  return B2_OK;
}

int gen_inputs(b2_plan* pl, void* d_in, int batch, uint64_t seed, cudaStream_t st) {
  const long n = (long)batch * pl->in_elems;
  if (pl->input_kind == B2_IN_TOKENS_I64) {
    CK(gen_tokens(static_cast<int64_t*>(d_in), n, pl->seq, (int)pl->in_elems, pl->vocab, seed,
                  st));
  } else {
    CK(gen_normal(static_cast<float*>(d_in), n, seed, st));
  }
  return B2_OK;
}

int check_device(b2_plan* pl) {
  int cur = -1;
  CK(cudaGetDevice(&cur));
  if (cur != pl->device) CK(cudaSetDevice(pl->device));
  return B2_OK;
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

const char* b2_last_error(void) { return g_err.c_str(); }

const char* b2_version(void) { return "libb2 0.1 sm_100a (tcgen05/TMA bf16, SIMT fp32)"; }

// INPUT (flat, unpadded) -> LINEAR -> LINEAR -> OUTPUT (only that tensor) with
// the hidden tensor consumed by the second linear alone: one mlp2 launch.
void plan_fuse_mlp(b2_plan* pl) {
  if (!pl->use_mlp_fusion || pl->force_simt || pl->layers.size() != 4) return;
  const Layer &I = pl->layers[0], &A = pl->layers[1], &Bl = pl->layers[2], &O = pl->layers[3];
  if (I.kind != OP_INPUT || A.kind != OP_LINEAR || Bl.kind != OP_LINEAR || O.kind != OP_OUTPUT)
    return;
  const int *pi = I.p, *pa = A.p, *pb = Bl.p, *po = O.p;
  if (pi[2] != 1 || pi[3] != 1 || pi[4] != pi[1]) return;             // flat input, no padding
  if (pa[0] != pi[0] || pa[6] != 1 || pa[8] >= 0 || pa[9] != pa[4]) return;
  if (pb[0] != pa[1] || pb[6] != 1 || pb[8] >= 0 || pb[9] != pb[4]) return;
  if (po[0] != 1 || po[1] != pb[1] || po[2] != 0) return;
  if (pa[4] != pi[1] || pb[4] != pa[5] || pa[4] > 2048 || pb[5] > 112 || pa[5] > 1024) return;
  // shared-memory staging (fp32 plans: hi + lo weight rows) and 16-byte bulk rows
  const size_t l1 = 2 * 16 * (size_t)pa[4] * 4 + (size_t)16 * pa[4] * 4;
  const size_t l2 = (16 + 2 * (size_t)pb[5]) * pa[5] * 4;
  if ((l1 > l2 ? l1 : l2) > 200 * 1024 || pa[4] % 8 || pa[5] % 8) return;
  pl->mlp_in = 0;
  pl->mlp_l1 = 1;
  pl->mlp_l2 = 2;
  pl->mlp_out = 3;
}

int b2_plan_create(const void* blob, size_t len, int dtype, b2_plan** out) {
  if (!blob || !out) return fail(B2_ERR_ARG, "null argument");
  *out = nullptr;
  const uint8_t* d = static_cast<const uint8_t*>(blob);
  if (len < sizeof(Header) + 4) return fail(B2_ERR_FORMAT, "truncated plan");
  Header h;
  memcpy(&h, d, sizeof h);
  if (memcmp(h.magic, "B2PL", 4) != 0) return fail(B2_ERR_FORMAT, "bad magic, not a b200-plan");
  if (h.version != 1) return fail(B2_ERR_FORMAT, "unsupported plan version %u", h.version);
  uint32_t crc;
  memcpy(&crc, d + len - 4, 4);
  if (crc32(d, len - 4) != crc) return fail(B2_ERR_FORMAT, "CRC mismatch, plan corrupted");
  const size_t tables = sizeof(Header) + (size_t)h.n_tensors * sizeof(TensorRec) +
                        (size_t)h.n_weights * sizeof(WeightRec) + (size_t)h.n_ops * sizeof(OpRec) +
                        h.meta_len;
  if (tables > len - 4) return fail(B2_ERR_FORMAT, "truncated plan tables");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(B2_ERR_NODEVICE, "no CUDA device visible");

  b2_plan* pl = new b2_plan();
  pl->dtype = dtype == B2_DT_FROM_PLAN ? (int)h.dtype : dtype;
  if (pl->dtype != B2_DT_FP32 && pl->dtype != B2_DT_BF16) {
    delete pl;
    return fail(B2_ERR_ARG, "dtype must be 0 (fp32) or 1 (bf16)");
  }
  pl->input_kind = (int)h.input_kind;
  pl->in_elems = h.in_elems;
  pl->out_elems = h.out_elems;
  // Developer knobs (kernel-variant A/B, profiling aids) are honoured only
  // with B2_DEV=1: a production process runs the default selection, the one
  // the parity tests check, whatever else its environment holds.
  const char* dev_env = getenv("B2_DEV");
  const bool dev = dev_env && dev_env[0] == '1';
  auto knob = [dev](const char* name) -> const char* { return dev ? getenv(name) : nullptr; };
  const char* fs = knob("B2_FORCE_SIMT");
  pl->force_simt = fs && fs[0] == '1';
  if (const char* em = knob("B2_EPI_MODE")) pl->epi_mode = atoi(em);
  if (const char* sg = knob("B2_STAGES")) pl->stages_override = atoi(sg);
  if (const char* gt = knob("B2_GEMM_TS")) pl->ts_debug = atoi(gt);
  if (const char* fb = knob("B2_FORCE_BN")) pl->force_bn = atoi(fb);
  if (const char* pd = knob("B2_PDL")) g_pdl = pd[0] != '0';
  if (const char* fk = knob("B2_FOLD_MAX_K")) pl->fold_max_k = atoi(fk);
  if (const char* ic = knob("B2_IM2COL")) pl->use_im2col = ic[0] != '0';
  if (const char* i8 = knob("B2_IM2COL8")) pl->im2col8 = i8[0] == '1';
  if (const char* sd = knob("B2_S2D")) pl->use_s2d = sd[0] != '0';
  if (const char* bd = knob("B2_BAND")) pl->use_band = bd[0] != '0';
  if (const char* pr = knob("B2_PAIR")) pl->use_pair = pr[0] != '0';
  if (const char* bp = knob("B2_BAND_PAIR")) pl->band_pair = bp[0] != '0';
  if (const char* nk = knob("B2_NARROW_K")) pl->narrow_k = nk[0] != '0';
  if (const char* vb = knob("B2_VERBOSE")) pl->verbose = vb[0] == '1';
  if (const char* pm = knob("B2_PAIR_MIN_M")) pl->pair_min_m = atol(pm);
  if (const char* pk = knob("B2_PAIR_MIN_K")) pl->pair_min_k = atoi(pk);
  if (const char* pf = knob("B2_POOL_FUSION")) pl->use_pool_fusion = pf[0] != '0';
  if (const char* tf = knob("B2_TF32")) pl->use_tf32 = tf[0] != '0';
  if (const char* tg = knob("B2_TF32_GATHER")) pl->tf32_gather = tg[0] != '0';
  if (const char* df = knob("B2_DS_FOLD")) pl->use_ds_fold = df[0] != '0';
  if (const char* ao = knob("B2_ALT_ORDER")) pl->alt_order = ao[0] != '0';
  if (const char* sk = knob("B2_SPLIT")) pl->use_split = sk[0] != '0';
  if (const char* cz = knob("B2_CHAIN")) pl->use_chain = cz[0] != '0';
  if (const char* cd = knob("B2_CHAIN_DS2")) pl->chain_ds2 = cd[0] != '0';
  if (const char* mf = knob("B2_MLP_FUSE")) pl->use_mlp_fusion = mf[0] != '0';
  if (const char* bm = knob("B2_BAND_MAX_N")) pl->band_max_n = atoi(bm);
  const auto tv0 = std::chrono::steady_clock::now();
  cudaFree(nullptr);   // context creation, timed separately under B2_VERBOSE
  const auto tv1 = std::chrono::steady_clock::now();
  cudaGetDevice(&pl->device);
  cudaDeviceGetAttribute(&pl->num_sms, cudaDevAttrMultiProcessorCount, pl->device);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, pl->device);
  if (major != 10 && pl->dtype == B2_DT_BF16 && !pl->force_simt) {
    delete pl;
    return fail(B2_ERR_NODEVICE, "bf16 tcgen05 path needs an sm_100 device (got sm_%d0)", major);
  }
  size_t pos = sizeof(Header);
  pl->tensors.resize(h.n_tensors);
  memcpy(pl->tensors.data(), d + pos, h.n_tensors * sizeof(TensorRec));
  pos += h.n_tensors * sizeof(TensorRec);
  std::vector<WeightRec> wr(h.n_weights);
  memcpy(wr.data(), d + pos, h.n_weights * sizeof(WeightRec));
  pos += h.n_weights * sizeof(WeightRec);
  pl->layers.resize(h.n_ops);
  for (uint32_t i = 0; i < h.n_ops; ++i) {
    OpRec r;
    memcpy(&r, d + pos, sizeof r);
    pos += sizeof r;
    pl->layers[i].kind = (int)r.kind;
    memcpy(pl->layers[i].p, r.p, sizeof r.p);
  }
  pos += h.meta_len;
  pos = (pos + 63) / 64 * 64;
  if (pos > len - 4) {
    delete pl;
    return fail(B2_ERR_FORMAT, "truncated weight data");
  }
  int rc = validate_ops(pl);
  if (!rc) plan_s2d(pl);
  if (!rc) plan_fuse_pool(pl);
  if (!rc) plan_fold_downsample(pl);
  if (!rc) plan_chain(pl);
  if (!rc) plan_fuse_mlp(pl);
  if (!rc) rc = upload_weights(pl, d + pos, wr, len - 4 - pos);
  if (!rc && pl->dtype == B2_DT_BF16) {
    std::vector<float> eye(256 * 256, 0.f);
    for (int i = 0; i < 256; ++i) eye[i * 256 + i] = 1.f;
    rc = upload_as<bf16>(pl, eye, &pl->identity);
    if (!rc) {
      std::vector<float> z(8192, 0.f);
      rc = upload_f32(pl, z.data(), z.size(), &pl->zero_bias);
    }
  }
  if (pl->verbose) {
    cudaDeviceSynchronize();
    const auto tv2 = std::chrono::steady_clock::now();
    fprintf(stderr, "b2: plan create: context %.3f s, weights %.3f s (%zu bytes of blob)\n",
            std::chrono::duration<double>(tv1 - tv0).count(),
            std::chrono::duration<double>(tv2 - tv1).count(), len);
  }
  // uploads and their zero-fills ran on the legacy default stream: complete
  // them before the plan's non-blocking stream can touch the weights
  if (cudaDeviceSynchronize() != cudaSuccess && !rc) rc = fail(B2_ERR_CUDA, "weight upload failed");
  if (pl->stage) {
    cudaFree(pl->stage);
    pl->stage = nullptr;
    pl->stage_bytes = 0;
  }
  if (!rc) {
    // algorithmic FLOPs (2 per MAC) of the contraction ops, with the model's
    // true input channels (an image stem reads 3 channels padded to 8)
    std::map<int, int> true_c;
    for (const Layer& L : pl->layers)
      if (L.kind == OP_INPUT) true_c[L.p[0]] = L.p[1];
    for (const Layer& L : pl->layers) {
      const int* p = L.p;
      const int cin = true_c.count(p[0]) ? std::min(p[6], true_c[p[0]]) : p[6];
      if (L.kind == OP_CONV) pl->flops += 2.0 * p[12] * p[13] * p[7] * p[8] * p[9] * cin;
      if (L.kind == OP_LINEAR) pl->flops += 2.0 * p[6] * p[5] * p[4];
      if (L.kind == OP_DWCONV) pl->flops += 2.0 * p[9] * p[10] * p[6] * p[12] * p[12];
      if (L.kind == OP_ATTENTION) pl->flops += 4.0 * p[2] * p[4] * p[4] * p[3];
    }
    if (cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking) != cudaSuccess)
      rc = fail(B2_ERR_CUDA, "cannot create stream");
  }
  if (rc) {
    b2_plan_destroy(pl);
    return rc;
  }
  *out = pl;
  return B2_OK;
}

int b2_plan_io(const b2_plan* pl, int64_t* in_elems, int* in_kind, int64_t* out_elems) {
  if (!pl) return fail(B2_ERR_ARG, "null plan");
  if (in_elems) *in_elems = pl->in_elems;
  if (in_kind) *in_kind = pl->input_kind;
  if (out_elems) *out_elems = pl->out_elems;
  return B2_OK;
}

int b2_plan_info(const b2_plan* pl, double* flops, double* wbytes, int* launches, int* dtype) {
  if (!pl) return fail(B2_ERR_ARG, "null plan");
  if (flops) *flops = pl->flops;
  if (wbytes) *wbytes = pl->weight_bytes;
  if (launches) {
    int n = 0;
    for (const Layer& L : pl->layers) n += L.kind == OP_OUTPUT ? L.p[0] : L.fused ? 0 : 1;
    *launches = n;
  }
  if (dtype) *dtype = pl->dtype;
  return B2_OK;
}

int b2_plan_memory(const b2_plan* pl, uint64_t* device_bytes) {
  if (!pl || !device_bytes) return fail(B2_ERR_ARG, "null argument");
  *device_bytes = pl->dev_bytes;
  return B2_OK;
}

int b2_forward(b2_plan* pl, const void* d_in, void* d_out, int batch, void* stream) {
  if (!pl || !d_in || !d_out) return fail(B2_ERR_ARG, "null argument");
  if (batch < 1) return fail(B2_ERR_ARG, "batch must be >= 1");
  int rc = check_device(pl);
  if (rc) return rc;
  BatchState* S;
  if ((rc = get_state(pl, batch, &S))) return rc;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : pl->stream;
  return enqueue(pl, *S, d_in, static_cast<float*>(d_out), st);
}

int b2_forward_host(b2_plan* pl, const void* h_in, void* h_out, int batch) {
  if (!pl || !h_in || !h_out) return fail(B2_ERR_ARG, "null argument");
  if (batch < 1) return fail(B2_ERR_ARG, "batch must be >= 1");
  int rc = check_device(pl);
  if (rc) return rc;
  BatchState* S;
  if ((rc = get_state(pl, batch, &S))) return rc;
  cudaGraphExec_t g;
  if ((rc = graph_of(pl, *S, &g))) return rc;
  NvtxRange range("b2.forward_host b=%d", batch);
  CK(cudaMemcpyAsync(S->d_in, h_in, in_bytes(pl, batch), cudaMemcpyHostToDevice, pl->stream));
  CK(cudaGraphLaunch(g, pl->stream));
  CK(cudaMemcpyAsync(h_out, S->d_out, (size_t)batch * pl->out_elems * 4, cudaMemcpyDeviceToHost,
                     pl->stream));
  CK(cudaStreamSynchronize(pl->stream));
  return B2_OK;
}

int b2_gen_input(b2_plan* pl, void* d_in, int batch, uint64_t seed, void* stream) {
  if (!pl || !d_in || batch < 1) return fail(B2_ERR_ARG, "bad argument");
  int rc = check_device(pl);
  if (rc) return rc;
  return gen_inputs(pl, d_in, batch, seed, stream ? static_cast<cudaStream_t>(stream) : pl->stream);
}

// End-to-end closed loop with host buffers, software-pipelined over three
// streams: H2D of step i (pinned host -> device buffer i%2) on s_h2d, the
// forward graph of buffer i%2 on the plan stream, D2H of step i's logits on
// s_d2h.  Events order buffer reuse (H2D i waits for forward i-2; forward i
// waits for H2D i and for D2H i-2).  Latency of step i = H2D start -> D2H end;
// completion = first H2D start -> D2H end of step i.  Every step still moves
// its full input and output across PCIe inside the timed region.
static int bench_e2e_pipelined(b2_plan* pl, BatchState* S, int warmup, int n, float* lat_ms,
                               float* completion_ms) {
  const int batch = S->batch;
  cudaGraphExec_t g[2];
  int rc;
  if ((rc = graph_of(pl, *S, &g[0])) || (rc = graph_of(pl, *S, &g[1], true))) return rc;
  const size_t ib = in_bytes(pl, batch), ob = (size_t)batch * pl->out_elems * 4;
  if (!S->h_out2) CK(cudaMallocHost(&S->h_out2, ob));
  if (!S->s_h2d) {
    CK(cudaStreamCreateWithFlags(&S->s_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&S->s_d2h, cudaStreamNonBlocking));
  }
  void* din[2] = {S->d_in, S->d_in2};
  float* dout[2] = {S->d_out, S->d_out2};
  void* hout[2] = {S->h_out, S->h_out2};
  cudaEvent_t in_done[2], fwd_done[2], out_done[2];
  for (int k = 0; k < 2; ++k) {
    CK(cudaEventCreateWithFlags(&in_done[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&fwd_done[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&out_done[k], cudaEventDisableTiming));
  }
  // start from a quiet device: earlier work on the plan stream (input gen) done
  CK(cudaStreamSynchronize(pl->stream));
  std::vector<cudaEvent_t> ev(2 * (size_t)n);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  bool used[2] = {false, false};
  for (int i = -warmup; i < n; ++i) {
    const int k = (i + warmup) & 1;
    if (used[k]) CK(cudaStreamWaitEvent(S->s_h2d, fwd_done[k], 0));
    if (i >= 0) CK(cudaEventRecord(ev[2 * i], S->s_h2d));
    CK(cudaMemcpyAsync(din[k], S->h_in, ib, cudaMemcpyHostToDevice, S->s_h2d));
    CK(cudaEventRecord(in_done[k], S->s_h2d));
    CK(cudaStreamWaitEvent(pl->stream, in_done[k], 0));
    if (used[k]) CK(cudaStreamWaitEvent(pl->stream, out_done[k], 0));
    CK(cudaGraphLaunch(g[k], pl->stream));
    CK(cudaEventRecord(fwd_done[k], pl->stream));
    CK(cudaStreamWaitEvent(S->s_d2h, fwd_done[k], 0));
    CK(cudaMemcpyAsync(hout[k], dout[k], ob, cudaMemcpyDeviceToHost, S->s_d2h));
    CK(cudaEventRecord(out_done[k], S->s_d2h));
    if (i >= 0) CK(cudaEventRecord(ev[2 * i + 1], S->s_d2h));
    used[k] = true;
  }
  CK(cudaStreamSynchronize(S->s_d2h));
  CK(cudaStreamSynchronize(pl->stream));
  for (int i = 0; i < n; ++i) {
    CK(cudaEventElapsedTime(&lat_ms[i], ev[2 * i], ev[2 * i + 1]));
    CK(cudaEventElapsedTime(&completion_ms[i], ev[0], ev[2 * i + 1]));
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k) {
    cudaEventDestroy(in_done[k]);
    cudaEventDestroy(fwd_done[k]);
    cudaEventDestroy(out_done[k]);
  }
  return B2_OK;
}

static int bench_impl(b2_plan* pl, int batch, int warmup, int n, uint64_t seed, float* lat_ms,
                      float* completion_ms, bool e2e) {
  if (!pl || !lat_ms || !completion_ms) return fail(B2_ERR_ARG, "null argument");
  if (batch < 1 || n < 1 || warmup < 0) return fail(B2_ERR_ARG, "bad batch/n/warmup");
  int rc = check_device(pl);
  if (rc) return rc;
  BatchState* S;
  if ((rc = get_state(pl, batch, &S))) return rc;
  cudaGraphExec_t g;
  if ((rc = graph_of(pl, *S, &g))) return rc;
  if ((rc = gen_inputs(pl, S->d_in, batch, seed, pl->stream))) return rc;
  NvtxRange range("b2.bench%s b=%d warmup=%d n=%d", e2e ? "_e2e" : "", batch, warmup, n);
  const size_t ib = in_bytes(pl, batch), ob = (size_t)batch * pl->out_elems * 4;
  if (e2e && !S->h_in) {
    CK(cudaMallocHost(&S->h_in, ib));
    CK(cudaMallocHost(&S->h_out, ob));
    CK(cudaMemcpyAsync(S->h_in, S->d_in, ib, cudaMemcpyDeviceToHost, pl->stream));
  }
  const char* pp = getenv("B2_E2E_PIPELINE");
  if (e2e && !(pp && pp[0] == '0')) return bench_e2e_pipelined(pl, S, warmup, n, lat_ms, completion_ms);
  const char* fl = getenv("B2_BENCH_FLUSH_L2");
  const bool flush = fl && fl[0] == '1';
  if (flush && !pl->flush_buf) {
    pl->flush_bytes = 256ull << 20;
    CK(cudaMalloc(&pl->flush_buf, pl->flush_bytes));
  }
  for (int i = 0; i < warmup; ++i) {
    if (e2e) CK(cudaMemcpyAsync(S->d_in, S->h_in, ib, cudaMemcpyHostToDevice, pl->stream));
    CK(cudaGraphLaunch(g, pl->stream));
    if (e2e) CK(cudaMemcpyAsync(S->h_out, S->d_out, ob, cudaMemcpyDeviceToHost, pl->stream));
  }
  std::vector<cudaEvent_t> ev(2 * (size_t)n);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  for (int i = 0; i < n; ++i) {
    if (flush) CK(flush_l2(pl->flush_buf, pl->flush_bytes, pl->stream));
    CK(cudaEventRecord(ev[2 * i], pl->stream));
    if (e2e) CK(cudaMemcpyAsync(S->d_in, S->h_in, ib, cudaMemcpyHostToDevice, pl->stream));
    CK(cudaGraphLaunch(g, pl->stream));
    if (e2e) CK(cudaMemcpyAsync(S->h_out, S->d_out, ob, cudaMemcpyDeviceToHost, pl->stream));
    CK(cudaEventRecord(ev[2 * i + 1], pl->stream));
  }
  CK(cudaStreamSynchronize(pl->stream));
  for (int i = 0; i < n; ++i) {
    CK(cudaEventElapsedTime(&lat_ms[i], ev[2 * i], ev[2 * i + 1]));
    CK(cudaEventElapsedTime(&completion_ms[i], ev[0], ev[2 * i + 1]));
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return B2_OK;
}

int b2_bench(b2_plan* pl, int batch, int warmup, int n, uint64_t seed, float* lat_ms,
             float* completion_ms) {
  return bench_impl(pl, batch, warmup, n, seed, lat_ms, completion_ms, false);
}

int b2_bench_e2e(b2_plan* pl, int batch, int warmup, int n, uint64_t seed, float* lat_ms,
                 float* completion_ms) {
  return bench_impl(pl, batch, warmup, n, seed, lat_ms, completion_ms, true);
}

int b2_profile_ops(b2_plan* pl, int batch, int iters, float* op_ms, int* n_ops, int* op_kinds) {
  if (!pl || !op_ms || !n_ops || batch < 1 || iters < 1) return fail(B2_ERR_ARG, "bad argument");
  int rc = check_device(pl);
  if (rc) return rc;
  BatchState* S;
  if ((rc = get_state(pl, batch, &S))) return rc;
  if ((rc = gen_inputs(pl, S->d_in, batch, 1234, pl->stream))) return rc;
  const size_t nl = pl->layers.size();
  std::vector<cudaEvent_t> ev(nl + 1);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  std::vector<double> acc(nl, 0.0);
  NvtxRange range("b2.profile_ops b=%d iters=%d", batch, iters);
  for (int it = 0; it <= iters; ++it) {   // iteration 0 is a warm-up
    if ((rc = run_forward(pl, *S, S->d_in, S->d_out, pl->stream, ev.data()))) return rc;
    CK(cudaEventRecord(ev[nl], pl->stream));
    CK(cudaStreamSynchronize(pl->stream));
    if (it == 0) continue;
    for (size_t i = 0; i < nl; ++i) {
      float ms;
      CK(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      acc[i] += ms;
    }
  }
  for (size_t i = 0; i < nl; ++i) {
    op_ms[i] = (float)(acc[i] / iters);
    if (op_kinds) op_kinds[i] = pl->layers[i].kind;
  }
  *n_ops = (int)nl;
  for (auto& e : ev) cudaEventDestroy(e);
  return B2_OK;
}

int b2_read_tensor(b2_plan* pl, int batch, int tensor, void* host_out, size_t bytes) {
  if (!pl || !host_out) return fail(B2_ERR_ARG, "null argument");
  if (tensor < 0 || tensor >= (int)pl->tensors.size()) return fail(B2_ERR_ARG, "bad tensor id");
  auto it = pl->states.find(batch);
  if (it == pl->states.end()) return fail(B2_ERR_ARG, "no forward has run at batch %d", batch);
  const size_t need = (size_t)batch * pl->tensors[tensor].elems * elem_size(pl, tensor);
  if (bytes < need) return fail(B2_ERR_ARG, "buffer too small (%zu < %zu)", bytes, need);
  if (pl->virt[tensor])
    return fail(B2_ERR_FUSED, "tensor %d is fused into its consumer (not materialised)", tensor);
  int rc = check_device(pl);
  if (rc) return rc;
  CK(cudaStreamSynchronize(pl->stream));
  for (const Layer& L : pl->layers) {
    if (L.kind != OP_INPUT || !L.s2d || L.p[0] != tensor) continue;
    // logical NHWC [B, H, W, Cpad] view of the space-to-depth storage
    const int H = L.p[2], W = L.p[3], Cp = L.p[4], H2 = L.s2d_H2, W2 = L.s2d_W2;
    std::vector<uint16_t> raw((size_t)batch * H2 * W2 * 16);
    CK(cudaMemcpy(raw.data(), it->second.act[tensor], raw.size() * 2, cudaMemcpyDeviceToHost));
    uint16_t* o = static_cast<uint16_t*>(host_out);
    for (int n = 0; n < batch; ++n)
      for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
          for (int c = 0; c < Cp; ++c) {
            const int yy = y + L.s2d_shift, xx = x + L.s2d_shift;
            const int q = ((yy & 1) * 2 + (xx & 1)) * 4 + c;
            o[(((size_t)n * H + y) * W + x) * Cp + c] =
                c < 4 ? raw[(((size_t)n * H2 + (yy >> 1)) * W2 + (xx >> 1)) * 16 + q] : 0;
          }
    return B2_OK;
  }
  CK(cudaMemcpy(host_out, it->second.act[tensor], need, cudaMemcpyDeviceToHost));
  return B2_OK;
}

void b2_plan_destroy(b2_plan* pl) {
  if (!pl) return;
  cudaSetDevice(pl->device);
  if (pl->stream) cudaStreamSynchronize(pl->stream);
  for (auto& kv : pl->states) {
    BatchState& S = kv.second;
    if (S.graph) cudaGraphExecDestroy(S.graph);
    cudaFree(S.arena);
    cudaFree(S.d_in);
    cudaFree(S.d_out);
    if (S.h_in) cudaFreeHost(S.h_in);
    if (S.h_out) cudaFreeHost(S.h_out);
    if (S.graph2) cudaGraphExecDestroy(S.graph2);
    if (S.ws) cudaFree(S.ws);
    if (S.mlp_ctr) cudaFree(S.mlp_ctr);
    if (S.col) cudaFree(S.col);
    if (S.d_in2) cudaFree(S.d_in2);
    if (S.d_out2) cudaFree(S.d_out2);
    if (S.h_out2) cudaFreeHost(S.h_out2);
    if (S.s_h2d) cudaStreamSynchronize(S.s_h2d), cudaStreamDestroy(S.s_h2d);
    if (S.s_d2h) cudaStreamSynchronize(S.s_d2h), cudaStreamDestroy(S.s_d2h);
  }
  for (void* p : pl->allocs) cudaFree(p);
  if (pl->flush_buf) cudaFree(pl->flush_buf);
  if (pl->stream) cudaStreamDestroy(pl->stream);
  delete pl;
}

}  // extern "C"
