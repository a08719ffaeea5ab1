// SIMT kernels of the executor: layout packing, depthwise conv, pools,
// LayerNorm, embedding+LN, attention, elementwise ops, output gather, the
// seeded input generator, and the fp32 GEMM/implicit-GEMM used by fp32 plans.
// Storage type T is float (fp32 plans) or bf16; arithmetic is fp32 throughout.
// HBM-bound kernels map consecutive threads to the contiguous channel / feature
// dimension so every warp access is coalesced.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace b2 {

static inline unsigned nblk(long n, int t) { return (unsigned)((n + t - 1) / t); }

// ------------------------------------------------------------------ fp32 GEMM
// 64x64 output tile, 256 threads x (4x4) outputs, K step 16; A gathered from
// the implicit im2col view when a.conv != 0.
template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const GemmSimtArgs a) {
  __shared__ float As[16][68];
  __shared__ float Bs[16][68];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const T* A = static_cast<const T*>(a.a);
  const T* Wt = static_cast<const T*>(a.w);
  // loader rows: element e = tid + i*256 -> row e>>4, k e&15 ; rows are tid>>4 + 16 i
  int li_img[4], li_ih[4], li_iw[4];
  bool li_ok[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + (tid >> 4) + 16 * i;
    li_ok[i] = m < a.M;
    li_img[i] = li_ih[i] = li_iw[i] = 0;
    if (a.conv && li_ok[i]) {
      const int img = m / a.OHW;
      const int rem = m - img * a.OHW;
      const int oh = rem / a.OW;
      li_img[i] = img;
      li_ih[i] = oh * a.stride - a.pad;
      li_iw[i] = (rem - oh * a.OW) * a.stride - a.pad;
    }
  }
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < a.K; k0 += 16) {
    const int kk = tid & 15;
    const int k = k0 + kk;
    int tap = 0, c = 0, r = 0, s = 0;
    if (a.conv && k < a.K) {
      tap = k / a.C;
      c = k - tap * a.C;
      r = tap / a.S;
      s = tap - r * a.S;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = (tid >> 4) + 16 * i;
      const int m = m0 + row;
      float v = 0.f;
      if (li_ok[i] && k < a.K) {
        if (a.conv) {
          const int ih = li_ih[i] + r, iw = li_iw[i] + s;
          if ((unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W)
            v = to_f(A[(((size_t)li_img[i] * a.H + ih) * a.W + iw) * a.C + c]);
        } else {
          v = to_f(A[(size_t)m * a.lda + k]);
        }
      }
      As[kk][row] = v;
      const int n = n0 + row;
      Bs[kk][row] = (n < a.N && k < a.K) ? to_f(Wt[(size_t)n * a.ldw + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[q][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[q][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const T* R = static_cast<const T*>(a.res);
  T* O = static_cast<T*>(a.out);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= a.N) continue;
      float v = acc[i][j];
      if (a.bias) v += a.bias[n];
      if (R) v += to_f(R[(size_t)m * a.N + n]);
      O[(size_t)m * a.N + n] = from_f<T>(act_apply(v, a.act));
    }
  }
}

template <typename T> cudaError_t gemm_simt(const GemmSimtArgs& a, cudaStream_t st) {
  dim3 grid(nblk(a.N, 64), nblk(a.M, 64));
  gemm_simt_kernel<T><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ packing
template <typename T>
__global__ void input_pack_kernel(const float* __restrict__ in, T* __restrict__ out, int B, int C,
                                  int HW, int Cp) {
  const long pix = (long)blockIdx.x * blockDim.x + threadIdx.x;   // over B*HW
  if (pix >= (long)B * HW) return;
  const long b = pix / HW, p = pix - b * HW;
  const float* src = in + b * C * (long)HW + p;
  T* dst = out + pix * Cp;
  for (int c = 0; c < Cp; ++c) dst[c] = from_f<T>(c < C ? __ldg(src + (long)c * HW) : 0.f);
}
template <typename T>
__global__ void vec_pack_kernel(const float* __restrict__ in, T* __restrict__ out, int B, int C,
                                int Cp) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)B * Cp) return;
  const long b = i / Cp, c = i - b * Cp;
  out[i] = from_f<T>(c < C ? in[b * C + c] : 0.f);
}
// bf16 images padded to 8 channels (VGG's 3-channel input for the CGW = 8 band
// conv): one 16-byte store per pixel instead of eight 2-byte stores (158 us at
// b=256 for 359 MB of traffic).
__global__ void input_pack8_kernel(const float* __restrict__ in, bf16* __restrict__ out, int B,
                                   int C, int HW) {
  const long pix = (long)blockIdx.x * blockDim.x + threadIdx.x;   // over B*HW
  if (pix >= (long)B * HW) return;
  const long b = pix / HW, p = pix - b * HW;
  const float* src = in + b * C * (long)HW + p;
  float v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = c < C ? __ldg(src + (long)c * HW) : 0.f;
  reinterpret_cast<uint4*>(out)[pix] = make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]),
                                                  pack_bf16x2(v[4], v[5]), pack_bf16x2(v[6], v[7]));
}

template <typename T>
cudaError_t input_pack(const float* in, T* out, int B, int C, int H, int W, int Cp,
                       cudaStream_t st) {
  if constexpr (sizeof(T) == 2) {
    if (Cp == 8 && C <= 8 && H * W > 1) {
      input_pack8_kernel<<<nblk((long)B * H * W, 256), 256, 0, st>>>(
          in, reinterpret_cast<bf16*>(out), B, C, H * W);
      return cudaGetLastError();
    }
  }
  if (H * W == 1)
    vec_pack_kernel<T><<<nblk((long)B * Cp, 256), 256, 0, st>>>(in, out, B, C, Cp);
  else
    input_pack_kernel<T><<<nblk((long)B * H * W, 256), 256, 0, st>>>(in, out, B, C, H * W, Cp);
  return cudaGetLastError();
}

// 2x2 space-to-depth pack for stride-2 stems: out[n][Y][X][q], q = (dy*2+dx)*4 + c,
// holds in[n][c][2Y+dy-shift][2X+dx-shift] (zero outside the image / for c >= C).
__global__ void input_pack_s2d_kernel(const float* __restrict__ in, bf16* __restrict__ out, int B,
                                      int C, int H, int W, int shift, int H2, int W2) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;   // over B*H2*W2
  if (i >= (long)B * H2 * W2) return;
  const int X = (int)(i % W2);
  const long t = i / W2;
  const int Y = (int)(t % H2);
  const long n = t / H2;
  uint32_t w[8];
#pragma unroll
  for (int qq = 0; qq < 8; ++qq) {
    float v2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = qq * 2 + h;
      const int c = q & 3, dx = (q >> 2) & 1, dy = q >> 3;
      const int y = 2 * Y + dy - shift, x = 2 * X + dx - shift;
      v2[h] = (c < C && (unsigned)y < (unsigned)H && (unsigned)x < (unsigned)W)
                  ? __ldg(in + ((n * C + c) * H + y) * (long)W + x)
                  : 0.f;
    }
    w[qq] = pack_bf16x2(v2[0], v2[1]);
  }
  uint4* o = reinterpret_cast<uint4*>(out + i * 16);
  o[0] = make_uint4(w[0], w[1], w[2], w[3]);
  o[1] = make_uint4(w[4], w[5], w[6], w[7]);
}
cudaError_t input_pack_s2d(const float* in, bf16* out, int B, int C, int H, int W, int shift,
                           int H2, int W2, cudaStream_t st) {
  input_pack_s2d_kernel<<<nblk((long)B * H2 * W2, 256), 256, 0, st>>>(in, out, B, C, H, W, shift,
                                                                      H2, W2);
  return cudaGetLastError();
}

__global__ void tokens_kernel(const int64_t* in, int32_t* out, long n, int S, int stride,
                              int vocab) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long b = i / S, j = i - b * S;
  long v = in[b * stride + j];
  v = v < 0 ? 0 : (v >= vocab ? vocab - 1 : v);
  out[i] = (int32_t)v;
}
// attention_mask [S] int64 per sample (after the ids) -> key-validity bits:
// one warp per 32 keys, bit l of the word = key (w * 32 + l) attends
__global__ void keymask_kernel(const int64_t* in, uint32_t* out, int B, int S, int stride) {
  const int nw = (S + 31) / 32;
  const long wi = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wi >= (long)B * nw) return;
  const long b = wi / nw;
  const int key = (int)(wi - b * nw) * 32 + lane;
  const bool valid = key < S && in[b * stride + S + key] != 0;
  const uint32_t bits = __ballot_sync(0xffffffffu, valid);
  if (lane == 0) out[wi] = bits;
}
cudaError_t tokens_pack(const int64_t* in, int32_t* out, uint32_t* mask, int B, int S,
                        int stride, int vocab, cudaStream_t st) {
  const long n = (long)B * S;
  tokens_kernel<<<nblk(n, 256), 256, 0, st>>>(in, out, n, S, stride, vocab);
  if (mask) {
    const long warps = (long)B * ((S + 31) / 32);
    keymask_kernel<<<nblk(warps * 32, 256), 256, 0, st>>>(in, mask, B, S, stride);
  }
  return cudaGetLastError();
}

template <typename T>
__global__ void convert_kernel(const float* src, T* dst, long n) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = from_f<T>(src[i]);
}
template <typename T> cudaError_t convert_f32(const float* src, T* dst, long n, cudaStream_t st) {
  convert_kernel<T><<<nblk(n, 256), 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ depthwise conv
// w_rsc: [R*R][C] (tap-major so a warp's channel loads coalesce)
template <typename T>
__global__ void dwconv_kernel(const T* __restrict__ x, const T* __restrict__ w,
                              const float* __restrict__ bias, T* __restrict__ y, int B, int H,
                              int W, int C, int R, int stride, int pad, int OH, int OW, int act) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)B * OH * OW * C;
  if (i >= total) return;
  const int c = (int)(i % C);
  long p = i / C;
  const int ow = (int)(p % OW);
  p /= OW;
  const int oh = (int)(p % OH);
  const long b = p / OH;
  float acc = bias ? bias[c] : 0.f;
  const int ih0 = oh * stride - pad, iw0 = ow * stride - pad;
  for (int r = 0; r < R; ++r) {
    const int ih = ih0 + r;
    if ((unsigned)ih >= (unsigned)H) continue;
    for (int s = 0; s < R; ++s) {
      const int iw = iw0 + s;
      if ((unsigned)iw >= (unsigned)W) continue;
      acc = fmaf(to_f(x[((b * H + ih) * W + iw) * C + c]), to_f(w[(r * R + s) * C + c]), acc);
    }
  }
  y[i] = from_f<T>(act_apply(acc, act));
}
// 16-byte vectors of channels: VEC = 8 (bf16) or 4 (fp32) channels per thread
template <typename T> struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
  union {
    uint4 u;
    T e[16 / sizeof(T)];
  };
};

template <typename T>
__global__ void dwconv_vec_kernel(const T* __restrict__ x, const T* __restrict__ w,
                                  const float* __restrict__ bias, T* __restrict__ y, int B,
                                  int H, int W, int C, int R, int stride, int pad, int OH, int OW,
                                  int act) {
  constexpr int V = Vec16<T>::N;
  const int CV = C / V;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)B * OH * OW * CV;
  if (i >= total) return;
  const int cv = (int)(i % CV);
  long p = i / CV;
  const int ow = (int)(p % OW);
  p /= OW;
  const int oh = (int)(p % OH);
  const long b = p / OH;
  const int c0 = cv * V;
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = bias ? bias[c0 + k] : 0.f;
  const int ih0 = oh * stride - pad, iw0 = ow * stride - pad;
  for (int r = 0; r < R; ++r) {
    const int ih = ih0 + r;
    if ((unsigned)ih >= (unsigned)H) continue;
    for (int s = 0; s < R; ++s) {
      const int iw = iw0 + s;
      if ((unsigned)iw >= (unsigned)W) continue;
      Vec16<T> xv, wv;
      xv.u = __ldg(reinterpret_cast<const uint4*>(x + ((b * H + ih) * W + iw) * C + c0));
      wv.u = __ldg(reinterpret_cast<const uint4*>(w + (r * R + s) * C + c0));
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] = fmaf(to_f(xv.e[k]), to_f(wv.e[k]), acc[k]);
    }
  }
  Vec16<T> ov;
#pragma unroll
  for (int k = 0; k < V; ++k) ov.e[k] = from_f<T>(act_apply(acc[k], act));
  *reinterpret_cast<uint4*>(y + ((b * OH + oh) * OW + ow) * (long)C + c0) = ov.u;
}

// 3x3 depthwise (MobileNetV2), stride 1 or 2, pad 1: the nine 16-byte input
// loads and nine weight loads are all issued before any FMA (clamped
// addresses, out-of-image taps masked), activation and stride compile-time.
// The generic kernel's per-tap bounds branches serialised the loads.
// (A strip-mined variant with a sliding 3-row register window — 3 loads per
// output instead of 9 — measured slower: less parallelism, serial loads.)
template <typename T, int STRIDE, int ACT>
__global__ void __launch_bounds__(256) dwconv3_vec_kernel(const T* __restrict__ x,
                                                          const T* __restrict__ w,
                                                          const float* __restrict__ bias,
                                                          T* __restrict__ y, int B, int H, int W,
                                                          int C, int OH, int OW) {
  constexpr int V = Vec16<T>::N;
  const int CV = C / V;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)B * OH * OW * CV;
  if (i >= total) return;
  const int cv = (int)(i % CV);
  long p = i / CV;
  const int ow = (int)(p % OW);
  p /= OW;
  const int oh = (int)(p % OH);
  const long b = p / OH;
  const int c0 = cv * V;
  Vec16<T> xv[9], wv[9];
  bool ok[9];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int ih = oh * STRIDE - 1 + r;
    const int ihc = min(max(ih, 0), H - 1);
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int iw = ow * STRIDE - 1 + s;
      const int iwc = min(max(iw, 0), W - 1);
      ok[r * 3 + s] = (unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W;
      xv[r * 3 + s].u = __ldg(reinterpret_cast<const uint4*>(x + ((b * H + ihc) * W + iwc) * C + c0));
      wv[r * 3 + s].u = __ldg(reinterpret_cast<const uint4*>(w + (r * 3 + s) * C + c0));
    }
  }
  float acc[V];
  if (bias) {
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = __ldg(bias + c0 + k);
  } else {
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = 0.f;
  }
#pragma unroll
  for (int t = 0; t < 9; ++t)
#pragma unroll
    for (int k = 0; k < V; ++k)
      acc[k] = ok[t] ? fmaf(to_f(xv[t].e[k]), to_f(wv[t].e[k]), acc[k]) : acc[k];
  Vec16<T> ov;
#pragma unroll
  for (int k = 0; k < V; ++k) ov.e[k] = from_f<T>(act_t<ACT>(acc[k]));
  *reinterpret_cast<uint4*>(y + ((b * OH + oh) * OW + ow) * (long)C + c0) = ov.u;
}

// acc + x[k] * w[k] for element k of two 16-byte vectors. bf16 uses the
// mixed-precision FMA (fma.rn.f32.bf16 -> FHFMA.BF16 with .H1 half selects):
// bf16 x bf16 is exact in fp32, so this equals fmaf on the widened values but
// needs no conversion instructions.
template <typename T> struct DwFma;
template <> struct DwFma<float> {
  static B2_DEV float f(const Vec16<float>& x, const Vec16<float>& w, int k, float acc) {
    return fmaf(x.e[k], w.e[k], acc);
  }
};
template <> struct DwFma<bf16> {
  static B2_DEV float f(const Vec16<bf16>& x, const Vec16<bf16>& w, int k, float acc) {
    const uint32_t xs = (&x.u.x)[k >> 1], ws = (&w.u.x)[k >> 1];
    unsigned short xl, xh, wl, wh;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(xl), "=h"(xh) : "r"(xs));
    asm("mov.b32 {%0,%1}, %2;" : "=h"(wl), "=h"(wh) : "r"(ws));
    float d;
    if (k & 1)
      asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(xh), "h"(wh), "f"(acc));
    else
      asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(xl), "h"(wl), "f"(acc));
    return d;
  }
};

// Row-strip variant: one thread = one 16-byte channel vector x OWT adjacent
// outputs of one row. The 9 filter taps stay in registers for the strip and
// each input column is loaded once per filter row for all OWT outputs, so L1
// traffic per output drops from 18 to (3*(STRIDE*(OWT-1)+3) + 9) / OWT vectors.
// Index math is 32-bit (the flat kernel's 64-bit divides were most of its
// instruction stream). Out-of-image rows are skipped; strips touching the left
// or right image edge take a clamped, zero-filled load path.
template <typename T, int STRIDE, int ACT, int OWT>
__global__ void __launch_bounds__(256) dwconv3_strip_kernel(const T* __restrict__ x,
                                                            const T* __restrict__ w,
                                                            const float* __restrict__ bias,
                                                            T* __restrict__ y, int B, int H, int W,
                                                            int C, int OH, int OW, int NS) {
  constexpr int V = Vec16<T>::N;
  constexpr int IW = STRIDE * (OWT - 1) + 3;
  const int CV = C / V;
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (unsigned)(B * OH * NS * CV)) return;
  const int cv = (int)(i % (unsigned)CV);
  const unsigned rest = i / (unsigned)CV;
  const int strip = (int)(rest % (unsigned)NS);
  const unsigned row = rest / (unsigned)NS;   // b * OH + oh
  const int oh = (int)(row % (unsigned)OH);
  const int b = (int)(row / (unsigned)OH);
  const int c0 = cv * V;
  const int ow0 = strip * OWT;
  const int iw0 = ow0 * STRIDE - 1;
  const bool interior = iw0 >= 0 && iw0 + IW <= W;
  float acc[OWT][V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const float bv = bias ? __ldg(bias + c0 + k) : 0.f;
#pragma unroll
    for (int o = 0; o < OWT; ++o) acc[o][k] = bv;
  }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int ih = oh * STRIDE - 1 + r;
    if ((unsigned)ih >= (unsigned)H) continue;
    Vec16<T> wv[3];
#pragma unroll
    for (int s = 0; s < 3; ++s)
      wv[s].u = __ldg(reinterpret_cast<const uint4*>(w + (r * 3 + s) * C + c0));
    const T* xrow = x + ((size_t)(b * H + ih) * W) * C + c0;
    Vec16<T> xv[IW];
    if (interior) {
      const uint4* p = reinterpret_cast<const uint4*>(xrow + (size_t)iw0 * C);
      const int cs = C / V;   // uint4 stride between columns
#pragma unroll
      for (int j = 0; j < IW; ++j) xv[j].u = __ldg(p + j * cs);
    } else {
#pragma unroll
      for (int j = 0; j < IW; ++j) {
        const int iw = iw0 + j;
        const int iwc = min(max(iw, 0), W - 1);
        xv[j].u = __ldg(reinterpret_cast<const uint4*>(xrow + (size_t)iwc * C));
        if ((unsigned)iw >= (unsigned)W) xv[j].u = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int j = 0; j < IW; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k)
#pragma unroll
        for (int o = 0; o < OWT; ++o) {
          const int s = j - o * STRIDE;
          if (s >= 0 && s < 3) acc[o][k] = DwFma<T>::f(xv[j], wv[s], k, acc[o][k]);
        }
  }
  T* yrow = y + ((size_t)row * OW + ow0) * C + c0;
#pragma unroll
  for (int o = 0; o < OWT; ++o) {
    if (ow0 + o >= OW) break;
    if constexpr (sizeof(T) == 2) {   // pack pairs, ReLU / ReLU6 on packed bf16 (act_pack2)
      uint32_t w4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) w4[k] = act_pack2<ACT>(acc[o][2 * k], acc[o][2 * k + 1]);
      *reinterpret_cast<uint4*>(yrow + (size_t)o * C) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    } else {
      Vec16<T> ov;
#pragma unroll
      for (int k = 0; k < V; ++k) ov.e[k] = from_f<T>(act_t<ACT>(acc[o][k]));
      *reinterpret_cast<uint4*>(yrow + (size_t)o * C) = ov.u;
    }
  }
}

// Strip width (measured on MobileNetV2 b=256: stride 1 best at 8 when the row
// splits into whole strips of 8 (or is short), else 4; stride 2 best at 2;
// B2_DW_OWT / B2_DW_OWT2 override, 1 = the flat per-output kernel)
static int dw_owt(int stride, int OW) {
  // read per launch (not cached): launches are captured into CUDA graphs, so
  // this runs once per plan state, and tests switch widths within a process
  const char* dv = getenv("B2_DEV");
  const char* e = dv && dv[0] == '1' ? getenv(stride == 1 ? "B2_DW_OWT" : "B2_DW_OWT2") : nullptr;
  const int v = e ? atoi(e) : 0;
  if (v) return v;
  if (stride == 1) return (OW % 8 == 0 || OW < 16) ? 8 : 4;
  return 2;
}

template <typename T, int STRIDE, int OWT>
static cudaError_t dwconv3_strip_launch(const T* x, const T* w, const float* bias, T* y, int B,
                                        int H, int W, int C, int OH, int OW, int act,
                                        cudaStream_t st) {
  const int NS = (OW + OWT - 1) / OWT;
  const long total = (long)B * OH * NS * (C / Vec16<T>::N);
  switch (act) {
#define B2_DW3S(A)                                                                             \
  case A:                                                                                      \
    dwconv3_strip_kernel<T, STRIDE, A, OWT><<<nblk(total, 256), 256, 0, st>>>(            \
        x, w, bias, y, B, H, W, C, OH, OW, NS);                                                \
    return cudaGetLastError();
    B2_DW3S(ACT_NONE)
    B2_DW3S(ACT_RELU)
    B2_DW3S(ACT_RELU6)
#undef B2_DW3S
    default: return cudaErrorInvalidValue;
  }
}

template <typename T, int STRIDE>
static cudaError_t dwconv3_launch(const T* x, const T* w, const float* bias, T* y, int B, int H,
                                  int W, int C, int OH, int OW, int act, cudaStream_t st) {
  const long total = (long)B * OH * OW * (C / Vec16<T>::N);
  switch (act) {
#define B2_DW3(A)                                                                          \
  case A:                                                                                  \
    dwconv3_vec_kernel<T, STRIDE, A><<<nblk(total, 256), 256, 0, st>>>(x, w, bias, y, B, H, W, C, \
                                                                       OH, OW);            \
    return cudaGetLastError();
    B2_DW3(ACT_NONE)
    B2_DW3(ACT_RELU)
    B2_DW3(ACT_RELU6)
#undef B2_DW3
    default: return cudaErrorInvalidValue;
  }
}

template <typename T>
cudaError_t dwconv(const T* x, const T* w, const float* bias, T* y, int B, int H, int W, int C,
                   int R, int stride, int pad, int OH, int OW, int act, cudaStream_t st) {
  if (C % Vec16<T>::N == 0 && R == 3 && pad == 1 && (stride == 1 || stride == 2) &&
      (act == ACT_NONE || act == ACT_RELU || act == ACT_RELU6)) {
    const int owt = dw_owt(stride, OW);
    const long rows = (long)B * OH * (C / Vec16<T>::N);
    if (stride == 1 && owt == 8 && rows * ((OW + 7) / 8) < (1L << 31))
      return dwconv3_strip_launch<T, 1, 8>(x, w, bias, y, B, H, W, C, OH, OW, act, st);
    if (stride == 1 && owt == 4 && rows * ((OW + 3) / 4) < (1L << 31))
      return dwconv3_strip_launch<T, 1, 4>(x, w, bias, y, B, H, W, C, OH, OW, act, st);
    if (stride == 2 && owt == 4 && rows * ((OW + 3) / 4) < (1L << 31))
      return dwconv3_strip_launch<T, 2, 4>(x, w, bias, y, B, H, W, C, OH, OW, act, st);
    if (owt == 2 && rows * ((OW + 1) / 2) < (1L << 31))
      return stride == 1
                 ? dwconv3_strip_launch<T, 1, 2>(x, w, bias, y, B, H, W, C, OH, OW, act, st)
                 : dwconv3_strip_launch<T, 2, 2>(x, w, bias, y, B, H, W, C, OH, OW, act, st);
  }
  if (C % Vec16<T>::N == 0 && R == 3 && pad == 1 && (stride == 1 || stride == 2) &&
      (act == ACT_NONE || act == ACT_RELU || act == ACT_RELU6))
    return stride == 1 ? dwconv3_launch<T, 1>(x, w, bias, y, B, H, W, C, OH, OW, act, st)
                       : dwconv3_launch<T, 2>(x, w, bias, y, B, H, W, C, OH, OW, act, st);
  if (C % Vec16<T>::N == 0) {
    const long total = (long)B * OH * OW * (C / Vec16<T>::N);
    dwconv_vec_kernel<T><<<nblk(total, 256), 256, 0, st>>>(x, w, bias, y, B, H, W, C, R, stride,
                                                           pad, OH, OW, act);
    return cudaGetLastError();
  }
  const long total = (long)B * OH * OW * C;
  dwconv_kernel<T><<<nblk(total, 256), 256, 0, st>>>(x, w, bias, y, B, H, W, C, R, stride, pad,
                                                     OH, OW, act);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ pools
template <typename T>
__global__ void maxpool_kernel(const T* __restrict__ x, T* __restrict__ y, int B, int H, int W,
                               int C, int k, int stride, int pad, int OH, int OW) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)B * OH * OW * C;
  if (i >= total) return;
  const int c = (int)(i % C);
  long p = i / C;
  const int ow = (int)(p % OW);
  p /= OW;
  const int oh = (int)(p % OH);
  const long b = p / OH;
  float m = -INFINITY;
  for (int r = 0; r < k; ++r) {
    const int ih = oh * stride - pad + r;
    if ((unsigned)ih >= (unsigned)H) continue;
    for (int s = 0; s < k; ++s) {
      const int iw = ow * stride - pad + s;
      if ((unsigned)iw >= (unsigned)W) continue;
      m = fmaxf(m, to_f(x[((b * H + ih) * W + iw) * C + c]));
    }
  }
  y[i] = from_f<T>(m);
}
template <typename T>
__global__ void maxpool_vec_kernel(const T* __restrict__ x, T* __restrict__ y, int B, int H,
                                   int W, int C, int k, int stride, int pad, int OH, int OW) {
  constexpr int V = Vec16<T>::N;
  const int CV = C / V;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)B * OH * OW * CV;
  if (i >= total) return;
  const int cv = (int)(i % CV);
  long p = i / CV;
  const int ow = (int)(p % OW);
  p /= OW;
  const int oh = (int)(p % OH);
  const long b = p / OH;
  float m[V];
#pragma unroll
  for (int q = 0; q < V; ++q) m[q] = -INFINITY;
  for (int r = 0; r < k; ++r) {
    const int ih = oh * stride - pad + r;
    if ((unsigned)ih >= (unsigned)H) continue;
    for (int s = 0; s < k; ++s) {
      const int iw = ow * stride - pad + s;
      if ((unsigned)iw >= (unsigned)W) continue;
      Vec16<T> v;
      v.u = __ldg(reinterpret_cast<const uint4*>(x + ((b * H + ih) * W + iw) * C + cv * V));
#pragma unroll
      for (int q = 0; q < V; ++q) m[q] = fmaxf(m[q], to_f(v.e[q]));
    }
  }
  Vec16<T> o;
#pragma unroll
  for (int q = 0; q < V; ++q) o.e[q] = from_f<T>(m[q]);
  reinterpret_cast<uint4*>(y)[i] = o.u;
}

// 3x3 / stride 2 / pad 1 (the ResNet stem pool): all nine 16-byte loads
// issued before any max (clamped addresses, out-of-window taps masked to
// -inf) so each thread keeps 144 B in flight; the generic kernel's per-tap
// bounds branches serialised them (3 TB/s measured).
template <typename T>
__global__ void maxpool3s2_vec_kernel(const T* __restrict__ x, T* __restrict__ y, int B, int H,
                                      int W, int C, int OH, int OW) {
  constexpr int V = Vec16<T>::N;
  const int CV = C / V;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long total = (long)B * OH * OW * CV;
  if (i >= total) return;
  const int cv = (int)(i % CV);
  long p = i / CV;
  const int ow = (int)(p % OW);
  p /= OW;
  const int oh = (int)(p % OH);
  const long b = p / OH;
  Vec16<T> v[9];
  bool ok[9];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int ih = oh * 2 - 1 + r;
    const int ihc = min(max(ih, 0), H - 1);
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int iw = ow * 2 - 1 + s;
      const int iwc = min(max(iw, 0), W - 1);
      ok[r * 3 + s] = (unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W;
      v[r * 3 + s].u =
          __ldg(reinterpret_cast<const uint4*>(x + ((b * H + ihc) * W + iwc) * C + cv * V));
    }
  }
  float m[V];
#pragma unroll
  for (int q = 0; q < V; ++q) m[q] = -INFINITY;
#pragma unroll
  for (int t = 0; t < 9; ++t)
#pragma unroll
    for (int q = 0; q < V; ++q) m[q] = ok[t] ? fmaxf(m[q], to_f(v[t].e[q])) : m[q];
  Vec16<T> o;
#pragma unroll
  for (int q = 0; q < V; ++q) o.e[q] = from_f<T>(m[q]);
  reinterpret_cast<uint4*>(y)[i] = o.u;
}

template <typename T>
cudaError_t maxpool(const T* x, T* y, int B, int H, int W, int C, int k, int stride, int pad,
                    int OH, int OW, cudaStream_t st) {
  if (C % Vec16<T>::N == 0 && k == 3 && stride == 2 && pad == 1) {
    const long tv = (long)B * OH * OW * (C / Vec16<T>::N);
    maxpool3s2_vec_kernel<T><<<nblk(tv, 256), 256, 0, st>>>(x, y, B, H, W, C, OH, OW);
    return cudaGetLastError();
  }
  if (C % Vec16<T>::N == 0) {
    const long tv = (long)B * OH * OW * (C / Vec16<T>::N);
    maxpool_vec_kernel<T><<<nblk(tv, 256), 256, 0, st>>>(x, y, B, H, W, C, k, stride, pad, OH,
                                                         OW);
    return cudaGetLastError();
  }
  const long total = (long)B * OH * OW * C;
  maxpool_kernel<T><<<nblk(total, 256), 256, 0, st>>>(x, y, B, H, W, C, k, stride, pad, OH, OW);
  return cudaGetLastError();
}

// Split-K epilogue: out = act(sum_s ws[s] + bias + res) in bf16, slices
// summed in split order (bit-reproducible), 8 outputs per thread.
template <int ACT>
__global__ void splitk_finalize_kernel(const float* __restrict__ ws, int nsplit,
                                       const float* __restrict__ bias,
                                       const bf16* __restrict__ res, bf16* __restrict__ out,
                                       long M, int N) {
  const long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i >= M * N) return;
  const int n = (int)(i % N);
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int sp = 0; sp < nsplit; ++sp) {
    const float4* w4 = reinterpret_cast<const float4*>(ws + (size_t)sp * M * N + i);
    const float4 a = __ldcg(w4), b = __ldcg(w4 + 1);
    v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
    v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
  }
  if (bias) {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] += __ldg(bias + n + e);
  }
  if (res) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(res + i));
    const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 f = unpack_bf16x2(rw[h]);
      v[2 * h] += f.x;
      v[2 * h + 1] += f.y;
    }
  }
  uint4 o;
  o.x = pack_bf16x2(act_t<ACT>(v[0]), act_t<ACT>(v[1]));
  o.y = pack_bf16x2(act_t<ACT>(v[2]), act_t<ACT>(v[3]));
  o.z = pack_bf16x2(act_t<ACT>(v[4]), act_t<ACT>(v[5]));
  o.w = pack_bf16x2(act_t<ACT>(v[6]), act_t<ACT>(v[7]));
  *reinterpret_cast<uint4*>(out + i) = o;
}

cudaError_t splitk_finalize(const float* ws, int nsplit, const float* bias, const bf16* res,
                            bf16* out, long M, int N, int act, cudaStream_t st) {
  if (N % 8 != 0) return cudaErrorInvalidValue;
  const long th = M * N / 8;
  switch (act) {
#define B2_SKF(A)                                                                              \
  case A:                                                                                      \
    splitk_finalize_kernel<A><<<nblk(th, 256), 256, 0, st>>>(ws, nsplit, bias, res, out, M, N); \
    return cudaGetLastError();
    B2_SKF(ACT_NONE)
    B2_SKF(ACT_RELU)
    B2_SKF(ACT_RELU6)
    B2_SKF(ACT_GELU)
    B2_SKF(ACT_TANH)
#undef B2_SKF
    default: return cudaErrorInvalidValue;
  }
}

template <typename T>
__global__ void avgpool_kernel(const T* __restrict__ x, T* __restrict__ y, int B, int HW, int C) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)B * C) return;
  const long b = i / C;
  const int c = (int)(i - b * C);
  const T* p = x + b * HW * (long)C + c;
  float s = 0.f;
  for (int q = 0; q < HW; ++q) s += to_f(p[(long)q * C]);
  y[i] = from_f<T>(s / HW);
}
// bf16, C % 8 == 0: a thread sums 8 channels with 16-byte loads (same per-channel
// order as the scalar kernel: bit-identical); the scalar version's 2-byte loads
// ran ResNet-50's 51 MB average pool at 2.9 TB/s
__global__ void avgpool8_kernel(const bf16* __restrict__ x, bf16* __restrict__ y, int B, int HW,
                                int C) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;   // over B * C / 8
  const int c8 = C / 8;
  if (i >= (long)B * c8) return;
  const long b = i / c8;
  const int c = (int)(i - b * c8) * 8;
  const bf16* p = x + b * HW * (long)C + c;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 7
  for (int q = 0; q < HW; ++q) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p + (long)q * C));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 f = unpack_bf16x2(w[h]);
      s[2 * h] += f.x;
      s[2 * h + 1] += f.y;
    }
  }
  uint32_t o[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) o[h] = pack_bf16x2(s[2 * h] / HW, s[2 * h + 1] / HW);
  reinterpret_cast<uint4*>(y + b * C + c)[0] = make_uint4(o[0], o[1], o[2], o[3]);
}

template <typename T>
cudaError_t avgpool(const T* x, T* y, int B, int HW, int C, cudaStream_t st) {
  if constexpr (sizeof(T) == 2) {
    if (C % 8 == 0) {
      avgpool8_kernel<<<nblk((long)B * C / 8, 128), 128, 0, st>>>(
          reinterpret_cast<const bf16*>(x), reinterpret_cast<bf16*>(y), B, HW, C);
      return cudaGetLastError();
    }
  }
  avgpool_kernel<T><<<nblk((long)B * C, 256), 256, 0, st>>>(x, y, B, HW, C);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ LayerNorm
B2_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one warp per row; rows of D <= 32*32 kept in registers
template <typename T>
__global__ void layernorm_kernel(const T* __restrict__ x, const T* __restrict__ res,
                                 const float* __restrict__ g, const float* __restrict__ bt,
                                 T* __restrict__ y, long rows, int D, float eps) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const T* xr = x + row * D;
  const T* rr = res ? res + row * D : nullptr;
  float v[32];
  const int per = (D + 31) / 32;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < per) {
      const int d = lane + 32 * i;
      float t = 0.f;
      if (d < D) {
        t = to_f(xr[d]);
        if (rr) t += to_f(rr[d]);
      }
      v[i] = t;
      s += t;
    }
  }
  const float mean = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < per) {
      const int d = lane + 32 * i;
      const float t = d < D ? v[i] - mean : 0.f;
      q += t * t;
    }
  }
  const float rstd = rsqrtf(warp_sum(q) / D + eps);
  T* yr = y + row * D;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < per) {
      const int d = lane + 32 * i;
      if (d < D) yr[d] = from_f<T>((v[i] - mean) * rstd * g[d] + bt[d]);
    }
  }
}
// bf16 rows with D % 256 == 0 (BERT D = 768): one warp per row, each lane
// moving 16-byte vectors (8 channels) — the scalar kernel's 2-byte loads ran
// at ~1/3 of HBM bandwidth.  Two-pass mean / variance in registers.
template <int VPL>
__global__ void __launch_bounds__(256) layernorm_vec_kernel(const bf16* __restrict__ x,
                                                            const bf16* __restrict__ res,
                                                            const float* __restrict__ g,
                                                            const float* __restrict__ bt,
                                                            bf16* __restrict__ y, long rows,
                                                            int D, float eps) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * D);
  const uint4* rr = res ? reinterpret_cast<const uint4*>(res + row * D) : nullptr;
  uint4 xv[VPL], rv[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    xv[i] = __ldg(xr + lane + 32 * i);
    rv[i] = rr ? __ldg(rr + lane + 32 * i) : make_uint4(0, 0, 0, 0);
  }
  float v[VPL][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const uint32_t xw[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
    const uint32_t rw[4] = {rv[i].x, rv[i].y, rv[i].z, rv[i].w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 a = unpack_bf16x2(xw[h]);
      const float2 b = unpack_bf16x2(rw[h]);
      v[i][2 * h] = a.x + b.x;
      v[i][2 * h + 1] = a.y + b.y;
      s += v[i][2 * h] + v[i][2 * h + 1];
    }
  }
  const float mean = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float t = v[i][e] - mean;
      q += t * t;
    }
  const float rstd = rsqrtf(warp_sum(q) / D + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + row * D);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int d0 = (lane + 32 * i) * 8;
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(g + d0));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(g + d0 + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(bt + d0));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(bt + d0 + 4));
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = (v[i][e] - mean) * rstd * gg[e] + bb[e];
    uint4 w;
    w.x = pack_bf16x2(o[0], o[1]);
    w.y = pack_bf16x2(o[2], o[3]);
    w.z = pack_bf16x2(o[4], o[5]);
    w.w = pack_bf16x2(o[6], o[7]);
    yr[lane + 32 * i] = w;
  }
}

// bf16 LayerNorm without a residual (BERT: the residual is added by the
// producing GEMM's epilogue), D = VPL * 256.  ncu on the one-row-per-warp
// kernel above: 15.3 us per BERT LayerNorm at b=128, issue-bound (IPC 1.74,
// ~17 instructions per element: gamma/beta reloaded for every row, scalar
// fp32 math) at 50% occupancy.  Here a warp keeps its lane's gamma/beta as
// f32x2 pairs in registers and walks rows r, r + nwarps, ... with the next
// row's 48 bytes per lane prefetched; sums, centring, scaling and the affine
// run on packed fma/mul/add.rn.f32x2 (FFMA2 ...): ~5 instructions per element.
B2_DEV uint64_t bf16x2_to_f2(uint32_t w) {   // (lo, hi) bf16 pair -> (f32, f32)
  return f2pack(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

template <int VPL>
__global__ void __launch_bounds__(256, 2) layernorm_rows_kernel(const bf16* __restrict__ x,
                                                                const float* __restrict__ g,
                                                                const float* __restrict__ bt,
                                                                bf16* __restrict__ y, long rows,
                                                                int D, float eps) {
  const int lane = threadIdx.x & 31;
  const long w0 = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long nw = (long)gridDim.x * (blockDim.x >> 5);
  if (w0 >= rows) return;
  uint64_t gg[VPL][4], bb[VPL][4];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const float4* gp = reinterpret_cast<const float4*>(g + (lane + 32 * i) * 8);
    const float4* bp = reinterpret_cast<const float4*>(bt + (lane + 32 * i) * 8);
    const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1), b0 = __ldg(bp), b1 = __ldg(bp + 1);
    gg[i][0] = f2pack(g0.x, g0.y);
    gg[i][1] = f2pack(g0.z, g0.w);
    gg[i][2] = f2pack(g1.x, g1.y);
    gg[i][3] = f2pack(g1.z, g1.w);
    bb[i][0] = f2pack(b0.x, b0.y);
    bb[i][1] = f2pack(b0.z, b0.w);
    bb[i][2] = f2pack(b1.x, b1.y);
    bb[i][3] = f2pack(b1.z, b1.w);
  }
  const float inv_d = 1.f / (float)D;
  // PDL: launched while the producing GEMM drains; gamma/beta (weights) are
  // read before the wait, the rows after it
  pdl_wait();
  pdl_launch_dependents();
  // rows r and r + nw in flight while row r is normalised (ncu: with one row
  // of prefetch the copy of the prefetched registers waited on DRAM, 25% of
  // the kernel's stall samples)
  uint4 cur[VPL], nxt[VPL];
  {
    const uint4* xr = reinterpret_cast<const uint4*>(x + w0 * D);
#pragma unroll
    for (int i = 0; i < VPL; ++i) cur[i] = __ldg(xr + lane + 32 * i);
    if (w0 + nw < rows) {
      const uint4* xn = reinterpret_cast<const uint4*>(x + (w0 + nw) * D);
#pragma unroll
      for (int i = 0; i < VPL; ++i) nxt[i] = __ldg(xn + lane + 32 * i);
    }
  }
  for (long r = w0; r < rows; r += nw) {
    uint4 nxt2[VPL];
    if (r + 2 * nw < rows) {
      const uint4* xr = reinterpret_cast<const uint4*>(x + (r + 2 * nw) * D);
#pragma unroll
      for (int i = 0; i < VPL; ++i) nxt2[i] = __ldg(xr + lane + 32 * i);
    }
    uint64_t v[VPL][4];
    uint64_t s2 = 0;   // (+0.f, +0.f)
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      v[i][0] = bf16x2_to_f2(cur[i].x);
      v[i][1] = bf16x2_to_f2(cur[i].y);
      v[i][2] = bf16x2_to_f2(cur[i].z);
      v[i][3] = bf16x2_to_f2(cur[i].w);
#pragma unroll
      for (int h = 0; h < 4; ++h) s2 = f2add(s2, v[i][h]);
    }
    float sa, sb;
    f2unpack(s2, sa, sb);
    const float mean = warp_sum(sa + sb) * inv_d;
    const uint64_t nm = f2pack(-mean, -mean);
    uint64_t q2 = 0;
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        v[i][h] = f2add(v[i][h], nm);          // centred
        q2 = f2fma(v[i][h], v[i][h], q2);
      }
    f2unpack(q2, sa, sb);
    const float rstd = rsqrtf(warp_sum(sa + sb) * inv_d + eps);
    const uint64_t rs = f2pack(rstd, rstd);
    uint4* yr = reinterpret_cast<uint4*>(y + r * D);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float oa, ob;
        f2unpack(f2fma(f2mul(v[i][h], rs), gg[i][h], bb[i][h]), oa, ob);
        o[h] = pack_bf16x2(oa, ob);
      }
      yr[lane + 32 * i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      cur[i] = nxt[i];
      nxt[i] = nxt2[i];
    }
  }
}

template <typename T>
cudaError_t layernorm(const T* x, const T* res, const float* g, const float* b, T* y, long rows,
                      int D, float eps, cudaStream_t st) {
  if (D > 1024) return cudaErrorInvalidValue;
  if constexpr (sizeof(T) == 2) {
    if (D % 256 == 0) {
      switch (D / 256) {
#define B2_LNV(V)                                                                           \
  case V:                                                                                   \
    if (!res) {                                                                             \
      static int sms = 0;                                                                   \
      if (!sms) {                                                                           \
        int dev = 0;                                                                        \
        cudaGetDevice(&dev);                                                                \
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);                  \
      }                                                                                     \
      const long blocks = (rows + 7) / 8;                                                   \
      return launch_pdl(layernorm_rows_kernel<V>,                                           \
                        dim3((unsigned)(blocks < 2 * sms ? blocks : 2 * sms)), dim3(256), 0, st, \
                        reinterpret_cast<const bf16*>(x), g, b, reinterpret_cast<bf16*>(y),  \
                        rows, D, eps);                                                      \
    }                                                                                       \
    layernorm_vec_kernel<V><<<nblk(rows, 8), 256, 0, st>>>(                                 \
        reinterpret_cast<const bf16*>(x), reinterpret_cast<const bf16*>(res), g, b,         \
        reinterpret_cast<bf16*>(y), rows, D, eps);                                          \
    return cudaGetLastError();
        B2_LNV(1)
        B2_LNV(2)
        B2_LNV(3)
        B2_LNV(4)
#undef B2_LNV
      }
    }
  }
  layernorm_kernel<T><<<nblk(rows, 8), 256, 0, st>>>(x, res, g, b, y, rows, D, eps);
  return cudaGetLastError();
}

template <typename T>
__global__ void embed_ln_kernel(const int32_t* __restrict__ ids, const T* __restrict__ word,
                                const T* __restrict__ pos, const T* __restrict__ type,
                                const float* __restrict__ g, const float* __restrict__ bt,
                                T* __restrict__ y, int B, int S, int D, float eps) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long)B * S) return;
  const int sidx = (int)(row % S);
  const long id = ids[row];
  float v[32];
  const int per = (D + 31) / 32;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < per) {
      const int d = lane + 32 * i;
      float t = 0.f;
      if (d < D) t = to_f(word[id * D + d]) + to_f(pos[(long)sidx * D + d]) + to_f(type[d]);
      v[i] = t;
      s += t;
    }
  }
  const float mean = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < per) {
      const int d = lane + 32 * i;
      const float t = d < D ? v[i] - mean : 0.f;
      q += t * t;
    }
  }
  const float rstd = rsqrtf(warp_sum(q) / D + eps);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < per) {
      const int d = lane + 32 * i;
      if (d < D) y[row * D + d] = from_f<T>((v[i] - mean) * rstd * g[d] + bt[d]);
    }
  }
}
// bf16, D % 256 == 0: one warp per token row on 16-byte vectors (8 channels
// per lane access), the three table rows loaded before any reduction; same
// two-pass mean / variance as the scalar kernel (whose 2-byte gathers ran the
// BERT embedding at under 0.5 TB/s).
template <int VPL>
__global__ void __launch_bounds__(256) embed_ln_vec_kernel(
    const int32_t* __restrict__ ids, const bf16* __restrict__ word, const bf16* __restrict__ pos,
    const bf16* __restrict__ type, const float* __restrict__ g, const float* __restrict__ bt,
    bf16* __restrict__ y, int B, int S, int D, float eps) {
  const long row = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long)B * S) return;
  const int sidx = (int)(row % S);
  const long id = ids[row];
  const uint4* wr = reinterpret_cast<const uint4*>(word + id * D);
  const uint4* pr = reinterpret_cast<const uint4*>(pos + (long)sidx * D);
  const uint4* tr = reinterpret_cast<const uint4*>(type);
  uint4 wv[VPL], pv[VPL], tv[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    wv[i] = __ldg(wr + lane + 32 * i);
    pv[i] = __ldg(pr + lane + 32 * i);
    tv[i] = __ldg(tr + lane + 32 * i);
  }
  float v[VPL][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const uint32_t a4[4] = {wv[i].x, wv[i].y, wv[i].z, wv[i].w};
    const uint32_t b4[4] = {pv[i].x, pv[i].y, pv[i].z, pv[i].w};
    const uint32_t c4[4] = {tv[i].x, tv[i].y, tv[i].z, tv[i].w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float2 a = unpack_bf16x2(a4[h]), b = unpack_bf16x2(b4[h]), c = unpack_bf16x2(c4[h]);
      v[i][2 * h] = a.x + b.x + c.x;
      v[i][2 * h + 1] = a.y + b.y + c.y;
      s += v[i][2 * h] + v[i][2 * h + 1];
    }
  }
  const float mean = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float t = v[i][e] - mean;
      q += t * t;
    }
  const float rstd = rsqrtf(warp_sum(q) / D + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + row * D);
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int d0 = (lane + 32 * i) * 8;
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(g + d0));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(g + d0 + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(bt + d0));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(bt + d0 + 4));
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = (v[i][e] - mean) * rstd * gg[e] + bb[e];
    uint4 w;
    w.x = pack_bf16x2(o[0], o[1]);
    w.y = pack_bf16x2(o[2], o[3]);
    w.z = pack_bf16x2(o[4], o[5]);
    w.w = pack_bf16x2(o[6], o[7]);
    yr[lane + 32 * i] = w;
  }
}

template <typename T>
cudaError_t embed_ln(const int32_t* ids, const T* word, const T* pos, const T* type,
                     const float* g, const float* b, T* y, int B, int S, int D, float eps,
                     cudaStream_t st) {
  if (D > 1024) return cudaErrorInvalidValue;
  if constexpr (sizeof(T) == 2) {
    if (D % 256 == 0) {
      const unsigned grid = nblk((long)B * S, 8);
      switch (D / 256) {
#define B2_ELV(V)                                                                            \
  case V:                                                                                    \
    embed_ln_vec_kernel<V><<<grid, 256, 0, st>>>(ids, word, pos, type, g, b, y, B, S, D, eps); \
    return cudaGetLastError();
        B2_ELV(1)
        B2_ELV(2)
        B2_ELV(3)
        B2_ELV(4)
#undef B2_ELV
      }
    }
  }
  embed_ln_kernel<T><<<nblk((long)B * S, 8), 256, 0, st>>>(ids, word, pos, type, g, b, y, B, S,
                                                          D, eps);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ attention
// One CTA per (sample, head); K and V of the head staged in shared memory as
// fp32; each thread owns query rows and runs a single-pass online softmax.
template <typename T, int DH>
__global__ void attention_kernel(const T* __restrict__ qkv, T* __restrict__ out, int S, int H,
                                 const uint32_t* __restrict__ keymask) {
  extern __shared__ float kv[];
  float* Ks = kv;
  float* Vs = kv + S * DH;
  const int b = blockIdx.x / H, h = blockIdx.x % H;
  const long ld = 3L * H * DH;
  const T* base = qkv + (long)b * S * ld;
  for (int i = threadIdx.x; i < S * DH; i += blockDim.x) {
    const int s = i / DH, d = i - s * DH;
    Ks[i] = to_f(base[s * ld + (long)H * DH + h * DH + d]);
    Vs[i] = to_f(base[s * ld + 2L * H * DH + h * DH + d]);
  }
  __syncthreads();
  const float scale = rsqrtf((float)DH);
  for (int qi = threadIdx.x; qi < S; qi += blockDim.x) {
    float q[DH], o[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) {
      q[d] = to_f(base[qi * ld + h * DH + d]) * scale;
      o[d] = 0.f;
    }
    float mx = -INFINITY, sum = 0.f;
    for (int j = 0; j < S; ++j) {
      float sc = 0.f;
#pragma unroll
      for (int d = 0; d < DH; ++d) sc = fmaf(q[d], Ks[j * DH + d], sc);
      if (keymask && !((keymask[(long)b * ((S + 31) / 32) + (j >> 5)] >> (j & 31)) & 1u))
        sc = -3.4028234663852886e38f;   // + float32 min (transformers' extended mask)
      if (sc > mx) {
        const float corr = __expf(mx - sc);
        sum *= corr;
#pragma unroll
        for (int d = 0; d < DH; ++d) o[d] *= corr;
        mx = sc;
      }
      const float p = __expf(sc - mx);
      sum += p;
#pragma unroll
      for (int d = 0; d < DH; ++d) o[d] = fmaf(p, Vs[j * DH + d], o[d]);
    }
    const float inv = 1.f / sum;
    T* orow = out + ((long)b * S + qi) * H * DH + h * DH;
#pragma unroll
    for (int d = 0; d < DH; ++d) orow[d] = from_f<T>(o[d] * inv);
  }
}
template <typename T>
cudaError_t attention(const T* qkv, T* out, int B, int S, int H, int Dh,
                      const uint32_t* keymask, cudaStream_t st) {
  if (Dh != 64) return cudaErrorInvalidValue;
  const size_t smem = (size_t)2 * S * 64 * sizeof(float);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(attention_kernel<T, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cfg = true;
  }
  attention_kernel<T, 64><<<B * H, 128, smem, st>>>(qkv, out, S, H, keymask);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ elementwise
template <typename T>
__global__ void act_kernel(const T* x, T* y, long n, int act) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = from_f<T>(act_apply(to_f(x[i]), act));
}
template <typename T> cudaError_t act_ew(const T* x, T* y, long n, int act, cudaStream_t st) {
  act_kernel<T><<<nblk(n, 256), 256, 0, st>>>(x, y, n, act);
  return cudaGetLastError();
}

template <typename T>
__global__ void output_gather_kernel(const T* src, float* out, int B, long elems, long ostride,
                                     long off) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)B * elems) return;
  const long b = i / elems, e = i - b * elems;
  out[b * ostride + off + e] = to_f(src[i]);
}
// 8 elements per thread: one 16-byte load (bf16) and two 16-byte stores.  The
// scalar kernel (a 64-bit division and a 2-byte load per element) took 40 us
// for BERT b=128's 25 MB sequence output (1.9 TB/s).
__global__ void output_gather8_kernel(const bf16* __restrict__ src, float* __restrict__ out,
                                      long n8, long elems8, long ostride, long off) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  const long b = i / elems8, e = (i - b * elems8) * 8;
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(src) + i);
  const float2 f0 = unpack_bf16x2(u.x), f1 = unpack_bf16x2(u.y), f2 = unpack_bf16x2(u.z),
               f3 = unpack_bf16x2(u.w);
  float4* o = reinterpret_cast<float4*>(out + b * ostride + off + e);
  o[0] = make_float4(f0.x, f0.y, f1.x, f1.y);
  o[1] = make_float4(f2.x, f2.y, f3.x, f3.y);
}

template <typename T>
cudaError_t output_gather(const T* src, float* out, int B, long elems, long ostride, long off,
                          cudaStream_t st) {
  if constexpr (sizeof(T) == 2) {
    if (elems % 8 == 0 && ostride % 4 == 0 && off % 4 == 0) {
      const long n8 = (long)B * elems / 8;
      output_gather8_kernel<<<nblk(n8, 256), 256, 0, st>>>(reinterpret_cast<const bf16*>(src),
                                                           out, n8, elems / 8, ostride, off);
      return cudaGetLastError();
    }
  }
  output_gather_kernel<T><<<nblk((long)B * elems, 256), 256, 0, st>>>(src, out, B, elems,
                                                                      ostride, off);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ input generator
// Counter-based: element i of stream `seed` -> splitmix64 -> Box-Muller.
// Restated on the CPU by oracle/gen_ref.py.
B2_DEV uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void gen_normal_kernel(float* out, long n, uint64_t seed) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t h = splitmix64(seed * 0xD1B54A32D192ED03ull + (uint64_t)i);
  const float u1 = ((float)(h >> 40) + 1.0f) * (1.0f / 16777216.0f);
  const float u2 = (float)((h >> 16) & 0xFFFFFFull) * (1.0f / 16777216.0f);
  out[i] = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}
// sample b = [ids(S), attention_mask(stride - S)]: id j hashes stream index
// b * S + j (the same ids as an unmasked plan); mask entries are 1
__global__ void gen_tokens_kernel(int64_t* out, long n, int S, int stride, int vocab,
                                  uint64_t seed) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long b = i / stride, j = i - b * stride;
  if (j >= S) {
    out[i] = 1;
    return;
  }
  const uint64_t h = splitmix64(seed * 0xD1B54A32D192ED03ull + (uint64_t)(b * S + j));
  out[i] = (int64_t)(((h >> 32) * (uint64_t)vocab) >> 32);
}
cudaError_t gen_normal(float* out, long n, uint64_t seed, cudaStream_t st) {
  gen_normal_kernel<<<nblk(n, 256), 256, 0, st>>>(out, n, seed);
  return cudaGetLastError();
}
cudaError_t gen_tokens(int64_t* out, long n, int S, int stride, int vocab, uint64_t seed,
                       cudaStream_t st) {
  gen_tokens_kernel<<<nblk(n, 256), 256, 0, st>>>(out, n, S, stride, vocab, seed);
  return cudaGetLastError();
}

__global__ void flush_kernel(uint4* p, long n, uint32_t v) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, v, v, v);
}
cudaError_t flush_l2(void* buf, size_t bytes, cudaStream_t st) {
  static uint32_t tick = 0;
  flush_kernel<<<148 * 4, 256, 0, st>>>(static_cast<uint4*>(buf), (long)(bytes / 16), ++tick);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ im2col (fp32)
// One thread per 4 consecutive K columns of one output pixel (a 16-byte store;
// kpad % 32 == 0): the 3-channel fp32 stems go to the 3xTF32 tensor-core GEMM
// over these rows instead of the FFMA conv (ResNet-50's fp32 stem was a
// quarter of the fp32 forward).
__global__ void im2col_f32_kernel(const float* __restrict__ x, float* __restrict__ col, long M,
                                  int H, int W, int C, int R, int S, int stride, int pad, int OH,
                                  int OW, int kpad) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int kq = kpad / 4;
  if (i >= M * kq) return;
  const long m = i / kq;
  const int k0 = (int)(i - m * kq) * 4;
  const int img = (int)(m / ((long)OH * OW));
  const int rem = (int)(m - (long)img * OH * OW);
  const int oh = rem / OW, ow = rem - oh * OW;
  const int K = R * S * C;
  float v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = k0 + j;
    v[j] = 0.f;
    if (k < K) {
      const int tap = k / C, c = k - tap * C;
      const int r = tap / S, s2 = tap - r * S;
      const int ih = oh * stride - pad + r, iw = ow * stride - pad + s2;
      if ((unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W)
        v[j] = __ldg(x + (((size_t)img * H + ih) * W + iw) * C + c);
    }
  }
  reinterpret_cast<float4*>(col)[i] = make_float4(v[0], v[1], v[2], v[3]);
}

cudaError_t im2col_f32(const float* x, float* col, int B, int H, int W, int C, int R, int S,
                       int stride, int pad, int OH, int OW, int kpad, cudaStream_t st) {
  const long M = (long)B * OH * OW;
  const long n = M * (kpad / 4);
  im2col_f32_kernel<<<nblk(n, 256), 256, 0, st>>>(x, col, M, H, W, C, R, S, stride, pad, OH, OW,
                                                   kpad);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ fused 2-layer MLP
// The reference's toy MLP (784 -> 256 -> act -> 10, BASELINE configs[0]) at
// batch 1..64 is launch-bound: input pack + two GEMMs + output gather were
// ~22 us per batch of graph replay for ~1 MB of weights.  One kernel instead:
// CTA (j, g) computes hidden units [16 j, 16 j + 16) for input rows
// [16 g, 16 g + 16) from its W1 slice and the rows staged in shared memory
// (input rounded to the plan's storage type, exactly like the packing op); the
// last CTA of a row group (arrival counter, reset by that CTA) computes the
// second layer for the group's rows in a fixed order and writes the logits
// tensor and the fp32 output.  Deterministic (every sum has one owner and one
// order).  fp32 plans keep their weights as the 3xTF32 hi + lo split, whose
// sum is the fp32 weight exactly.
constexpr int MLP_NB = 8, MLP_RB = 16;

// four consecutive storage elements as fp32 (8-byte bf16 / 16-byte fp32 loads)
template <typename T> B2_DEV float4 ld4f(const T* p);
template <> B2_DEV float4 ld4f<float>(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <> B2_DEV float4 ld4f<bf16>(const bf16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y);
  return make_float4(a.x, a.y, b.x, b.y);
}

// Rows [nrows][bytes] at a source pitch into shared memory at a destination
// pitch, one bulk copy per row, row r issued by thread `first + r` so the
// copies run concurrently (bulk copies issued by one thread complete one at a
// time, ~0.3 us each: serial issue made the staging 17 us).  A tiny MLP is
// latency-bound: the first version's element-wise staging loops paid one
// L2/DRAM round trip per few elements (73 us for a 2 MB problem).
B2_DEV void bulk_rows(void* dst, uint32_t dst_pitch, const void* src, size_t src_pitch, int nrows,
                      uint32_t bytes, uint64_t* bar, int first) {
  const int r = (int)threadIdx.x - first;
  if (r >= 0 && r < nrows)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(static_cast<uint8_t*>(dst) + (size_t)r * dst_pitch)),
        "l"(static_cast<const uint8_t*>(src) + (size_t)r * src_pitch), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <typename T>
__global__ void __launch_bounds__(256) mlp2_kernel(const MlpArgs a) {
  extern __shared__ __align__(16) uint8_t mraw[];
  const int K1 = a.K1, N1 = a.N1, N2 = a.N2;
  const bool split = a.w1lo != nullptr;              // fp32 plan: 3xTF32 hi + lo weights
  const uint32_t k1b = (uint32_t)K1 * sizeof(T), k1p = (k1b + 15) & ~15u;
  T* sw = reinterpret_cast<T*>(mraw);                // [16][k1p bytes] W1 slice (hi)
  T* swl = reinterpret_cast<T*>(mraw + MLP_NB * k1p);   // lo part (fp32 plans)
  float* sx = reinterpret_cast<float*>(mraw + (split ? 2 : 1) * MLP_NB * k1p);   // [16][K1]
  __shared__ uint64_t bar;
  __shared__ int last;
  __shared__ float sb2[256];
  const int n0 = blockIdx.x * MLP_NB, r0 = blockIdx.y * MLP_RB;
  const int rows = min(MLP_RB, a.B - r0), units = min(MLP_NB, N1 - n0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&bar, (uint32_t)(units * k1b * (split ? 2 : 1) + rows * K1 * 4));
  }
  __syncthreads();
  {
    const size_t wp = (size_t)a.ldw1 * sizeof(T);
    bulk_rows(sw, k1p, static_cast<const T*>(a.w1) + (size_t)n0 * a.ldw1, wp, units, k1b, &bar, 0);
    if (split)
      bulk_rows(swl, k1p, static_cast<const T*>(a.w1lo) + (size_t)n0 * a.ldw1, wp, units, k1b,
                &bar, 32);
    bulk_rows(sx, K1 * 4, a.in + (size_t)r0 * K1, (size_t)K1 * 4, rows, K1 * 4, &bar, 64);
  }
  mbar_wait(&bar, 0);
  // input rounded through the plan's storage type, like the packing op it replaces
  for (int e = threadIdx.x; e < rows * K1; e += blockDim.x) {
    const T xt = from_f<T>(sx[e]);
    sx[e] = to_f(xt);
    if (blockIdx.x == 0) static_cast<T*>(a.xin)[(size_t)r0 * K1 + e] = xt;
  }
  __syncthreads();
  // layer 1: warp = hidden unit, its 32 lanes split the K1-long dot in 4-wide
  // vectors (8- / 16-byte shared loads: element-wise loads made the dots
  // shared-memory-instruction bound), shuffle-reduced
  {
    const int n = threadIdx.x >> 5, kl = threadIdx.x & 31;
    const T* wr = reinterpret_cast<const T*>(reinterpret_cast<const uint8_t*>(sw) + n * k1p);
    const T* wl = reinterpret_cast<const T*>(reinterpret_cast<const uint8_t*>(swl) + n * k1p);
    const float bias1 = (a.b1 && n < units) ? __ldg(a.b1 + n0 + n) : 0.f;   // hoisted: an L2
    // round trip per row on the critical path cost more than the dots
    for (int r = 0; r < rows; ++r) {
      const float* xr = sx + r * K1;
      float acc = 0.f;
      if (n < units)
#pragma unroll 4
        for (int k = kl * 4; k < K1; k += 128) {
          float4 w = ld4f<T>(wr + k);
          if (split) {
            const float4 l = ld4f<T>(wl + k);
            w.x += l.x; w.y += l.y; w.z += l.z; w.w += l.w;
          }
          const float4 x = *reinterpret_cast<const float4*>(xr + k);
          acc = fmaf(x.x, w.x, fmaf(x.y, w.y, fmaf(x.z, w.z, fmaf(x.w, w.w, acc))));
        }
      acc = warp_sum(acc);
      if (kl == 0 && n < units) {
        acc += bias1;
        static_cast<T*>(a.h)[(size_t)(r0 + r) * N1 + n0 + n] = from_f<T>(act_apply(acc, a.act1));
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(a.counters + blockIdx.y, 1u);
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // layer 2 for this row group, by the last CTA to arrive: h rows (written by
  // the other CTAs of this launch; bulk copies read through L2) and W2
  __threadfence();
  asm volatile("fence.proxy.async.global;" ::: "memory");
  const uint32_t n1b = (uint32_t)N1 * sizeof(T), n1p = (n1b + 15) & ~15u;
  T* sh = reinterpret_cast<T*>(mraw);                                  // [rows][n1p bytes]
  T* sw2 = reinterpret_cast<T*>(mraw + MLP_RB * n1p);                  // [N2][n1p bytes]
  T* sw2l = reinterpret_cast<T*>(mraw + (MLP_RB + N2) * n1p);
  const bool split2 = a.w2lo != nullptr;
  if (threadIdx.x == 0)
    mbar_arrive_expect_tx(&bar, (uint32_t)(rows * n1b + N2 * n1b * (split2 ? 2 : 1)));
  __syncthreads();
  {
    const size_t wp = (size_t)a.ldw2 * sizeof(T);
    bulk_rows(sh, n1p, static_cast<const T*>(a.h) + (size_t)r0 * N1, n1b, rows, n1b, &bar, 0);
    bulk_rows(sw2, n1p, a.w2, wp, N2, n1b, &bar, 16);
    if (split2) bulk_rows(sw2l, n1p, a.w2lo, wp, N2, n1b, &bar, 16 + N2);
  }
  for (int m = threadIdx.x; m < N2; m += blockDim.x) sb2[m] = a.b2 ? __ldg(a.b2 + m) : 0.f;
  mbar_wait(&bar, 1);
  __syncthreads();
  // warp per output, lanes split the N1-long dot
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int o = warp; o < rows * N2; o += 8) {
    const int rr = o / N2, m = o - rr * N2;
    const T* hr = reinterpret_cast<const T*>(reinterpret_cast<const uint8_t*>(sh) + rr * n1p);
    const T* wr = reinterpret_cast<const T*>(reinterpret_cast<const uint8_t*>(sw2) + m * n1p);
    const T* wl = reinterpret_cast<const T*>(reinterpret_cast<const uint8_t*>(sw2l) + m * n1p);
    float acc = 0.f;
#pragma unroll 8
    for (int k = lane; k < N1; k += 32) {
      float w = to_f(wr[k]);
      if (split2) w += to_f(wl[k]);
      acc = fmaf(to_f(hr[k]), w, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      acc += sb2[m];
      const T yv = from_f<T>(act_apply(acc, a.act2));
      static_cast<T*>(a.y)[(size_t)(r0 + rr) * N2 + m] = yv;
      a.out[(size_t)(r0 + rr) * a.out_stride + a.out_off + m] = to_f(yv);
    }
  }
  if (threadIdx.x == 0) a.counters[blockIdx.y] = 0;   // ready for the next launch
}

template <typename T>
cudaError_t mlp2(const MlpArgs& a, cudaStream_t st) {
  const size_t k1p = ((size_t)a.K1 * sizeof(T) + 15) & ~size_t(15);
  const size_t n1p = ((size_t)a.N1 * sizeof(T) + 15) & ~size_t(15);
  const int sp = a.w1lo ? 2 : 1;
  const size_t l1 = sp * MLP_NB * k1p + (size_t)MLP_RB * a.K1 * 4;
  const size_t l2 = (MLP_RB + (size_t)a.N2 * sp) * n1p;
  const size_t smem = l1 > l2 ? l1 : l2;
  if ((a.K1 * sizeof(T)) % 16 || (a.N1 * sizeof(T)) % 16 || (a.ldw1 * sizeof(T)) % 16 ||
      (a.ldw2 * sizeof(T)) % 16 || (a.K1 * 4) % 16)
    return cudaErrorInvalidValue;   // bulk copies need 16-byte rows
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(mlp2_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cfg = true;
  }
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  dim3 grid((a.N1 + MLP_NB - 1) / MLP_NB, (a.B + MLP_RB - 1) / MLP_RB);
  mlp2_kernel<T><<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ instantiations
#define B2_INST(T)                                                                            \
  template cudaError_t gemm_simt<T>(const GemmSimtArgs&, cudaStream_t);                       \
  template cudaError_t input_pack<T>(const float*, T*, int, int, int, int, int, cudaStream_t); \
  template cudaError_t dwconv<T>(const T*, const T*, const float*, T*, int, int, int, int, int, \
                                 int, int, int, int, int, cudaStream_t);                       \
  template cudaError_t maxpool<T>(const T*, T*, int, int, int, int, int, int, int, int, int,   \
                                  cudaStream_t);                                               \
  template cudaError_t avgpool<T>(const T*, T*, int, int, int, cudaStream_t);                  \
  template cudaError_t layernorm<T>(const T*, const T*, const float*, const float*, T*, long,  \
                                    int, float, cudaStream_t);                                 \
  template cudaError_t embed_ln<T>(const int32_t*, const T*, const T*, const T*, const float*, \
                                   const float*, T*, int, int, int, float, cudaStream_t);      \
  template cudaError_t attention<T>(const T*, T*, int, int, int, int, const uint32_t*,      \
                                    cudaStream_t);           \
  template cudaError_t act_ew<T>(const T*, T*, long, int, cudaStream_t);                       \
  template cudaError_t output_gather<T>(const T*, float*, int, long, long, long, cudaStream_t); \
  template cudaError_t convert_f32<T>(const float*, T*, long, cudaStream_t);                  \
  template cudaError_t mlp2<T>(const MlpArgs&, cudaStream_t);
B2_INST(float)
B2_INST(bf16)
#undef B2_INST

}  // namespace b2
