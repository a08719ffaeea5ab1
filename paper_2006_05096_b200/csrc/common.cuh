// Shared device helpers for libb2 (sm_100a only): bf16 packing, mbarrier,
// TMA (cp.async.bulk.tensor), cp.async, and tcgen05 / TMEM wrappers written
// as inline PTX.  Descriptor encodings follow the sm_100 UMMA formats
// (shared-memory matrix descriptor: start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version=1 [46,48), layout [61,64); instruction descriptor:
// c_fmt [4,6), a_fmt [7,10), b_fmt [10,13), a/b major [15],[16], N>>3 [17,23),
// M>>4 [24,29)).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define B2_DEV __device__ __forceinline__

typedef __nv_bfloat16 bf16;

enum { ACT_NONE = 0, ACT_RELU = 1, ACT_RELU6 = 2, ACT_GELU = 3, ACT_TANH = 4 };

// GELU(x) = x/2 (1 + erf(x / sqrt 2)). (libdevice erff's branches made the
// GELU epilogue the bottleneck of the BERT FFN GEMM; A&S 7.1.26 needed two
// MUFU ops per element.)
// 1/x on the MUFU alone (__fdividef adds an FMUL and a range test + select:
// 3 of the ~20 instructions per element of the GELU epilogue)
B2_DEV float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
B2_DEV float gelu_erf(float v) {
  // erf by Abramowitz & Stegun 7.1.28: 1 - (1 + a1 z + ... + a6 z^6)^-16,
  // |error| <= 3e-7 (GELU within 1.1e-6 of the exact erf form over [-12, 12],
  // checked on the host). One MUFU (the reciprocal) per element instead of the
  // two (reciprocal + exp) of 7.1.26: the GELU epilogue of BERT's FFN GEMM is
  // MUFU-throughput bound (16 per clock per SM).
  const float z = fabsf(v) * 0.70710678118654752f;
  const float p = fmaf(z, fmaf(z, fmaf(z, fmaf(z, fmaf(z, fmaf(z, 0.0000430638f, 0.0002765672f),
                                                       0.0001520143f), 0.0092705272f),
                                         0.0422820123f), 0.0705230784f), 1.f);
  float r = rcp_approx(p);
  r *= r;
  r *= r;
  r *= r;
  r *= r;
  return 0.5f * v * (1.f + copysignf(1.f - r, v));
}

// Two GELUs on packed fp32 pairs (Blackwell FFMA2 / FMUL2 via fma.rn.f32x2 /
// mul.rn.f32x2): the same A&S 7.1.28 arithmetic as gelu_erf, per-lane
// identical results (f32x2 ops round each lane exactly like the scalar op),
// at about half the issue slots -- the BERT FFN GEMM epilogue is issue-bound.
B2_DEV uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
B2_DEV void f2unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
B2_DEV uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
B2_DEV uint64_t f2mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
B2_DEV uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// accumulator pair (raw tcgen05.ld words) + bias pair on one add.rn.f32x2
// (per-lane identical to the two scalar adds; half the issue slots)
B2_DEV float2 acc_add2(uint32_t a0, uint32_t a1, float b0, float b1) {
  float x, y;
  f2unpack(f2add(f2pack(__uint_as_float(a0), __uint_as_float(a1)), f2pack(b0, b1)), x, y);
  return make_float2(x, y);
}
B2_DEV void gelu_erf2(float& va, float& vb) {
  const float c = 0.70710678118654752f;
  const uint64_t z = f2pack(fabsf(va) * c, fabsf(vb) * c);
  uint64_t p = f2fma(z, f2pack(0.0000430638f, 0.0000430638f), f2pack(0.0002765672f, 0.0002765672f));
  p = f2fma(z, p, f2pack(0.0001520143f, 0.0001520143f));
  p = f2fma(z, p, f2pack(0.0092705272f, 0.0092705272f));
  p = f2fma(z, p, f2pack(0.0422820123f, 0.0422820123f));
  p = f2fma(z, p, f2pack(0.0705230784f, 0.0705230784f));
  p = f2fma(z, p, f2pack(1.f, 1.f));
  float pa, pb;
  f2unpack(p, pa, pb);
  uint64_t r = f2pack(rcp_approx(pa), rcp_approx(pb));
  r = f2mul(r, r);
  r = f2mul(r, r);
  r = f2mul(r, r);
  r = f2mul(r, r);
  float ra, rb;   // 1 - r as one packed fma (single rounding, same as the scalar subtract)
  f2unpack(f2fma(r, f2pack(-1.f, -1.f), f2pack(1.f, 1.f)), ra, rb);
  const float ea = copysignf(ra, va), eb = copysignf(rb, vb);
  const uint64_t h = f2mul(f2pack(va, vb), f2pack(0.5f, 0.5f));
  float oa, ob;
  f2unpack(f2fma(h, f2pack(ea, eb), h), oa, ob);
  va = oa;
  vb = ob;
}

B2_DEV float act_apply(float v, int act) {
  switch (act) {
    case ACT_RELU: return fmaxf(v, 0.f);
    case ACT_RELU6: return fminf(fmaxf(v, 0.f), 6.f);
    case ACT_GELU: return gelu_erf(v);
    case ACT_TANH: return tanhf(v);
    default: return v;
  }
}

template <int ACT> B2_DEV float act_t(float v) {
  if constexpr (ACT == ACT_RELU) return fmaxf(v, 0.f);
  else if constexpr (ACT == ACT_RELU6) return fminf(fmaxf(v, 0.f), 6.f);
  else if constexpr (ACT == ACT_GELU) return gelu_erf(v);
  else if constexpr (ACT == ACT_TANH) return tanhf(v);
  else return v;
}

template <typename T> B2_DEV float to_f(T v);
template <> B2_DEV float to_f<float>(float v) { return v; }
template <> B2_DEV float to_f<bf16>(bf16 v) { return __bfloat162float(v); }
template <typename T> B2_DEV T from_f(float v);
template <> B2_DEV float from_f<float>(float v) { return v; }
template <> B2_DEV bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

B2_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
B2_DEV float2 unpack_bf16x2(uint32_t v) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&v);
  return __bfloat1622float2(h);
}

// Activation + bf16 pack of a pair.  ReLU / ReLU6 are applied AFTER the
// round-to-nearest pack, on packed bf16 (max / min.bf16x2): rounding is
// monotone and 0 / 6 are exact in bf16, so the values equal act-then-round
// (only the sign of a zero may differ); one packed op instead of two scalar.
template <int ACT> B2_DEV uint32_t act_pack2(float a, float b) {
  if constexpr (ACT == ACT_RELU || ACT == ACT_RELU6) {
    uint32_t w = pack_bf16x2(a, b), d;
    if constexpr (ACT == ACT_RELU6) {
      asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(w), "r"(0x40C040C0u));   // 6.0, 6.0
      w = d;
    }
    asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(w), "r"(0u));
    return d;
  } else {
    return pack_bf16x2(act_t<ACT>(a), act_t<ACT>(b));
  }
}

B2_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
B2_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
B2_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
B2_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
B2_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
B2_DEV bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Spin on an mbarrier phase.  A watchdog turns a pipeline deadlock into a
// reported error (printf + trap -> cudaErrorLaunchFailure) after ~2^34 cycles
// instead of a hung GPU.
B2_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(a, parity)) {
    if (clock64() - t0 > (1ll << 34)) {
      printf("b2: mbarrier wait timeout (smem 0x%x parity %u) block %d thread %d\n", a, parity,
             blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}

// Address-based forms for producer loops that keep shared addresses as plain
// 32-bit values (no generic->shared conversion per K block).
B2_DEV void mbar_wait_u32(uint32_t a, uint32_t parity) {
  if (mbar_try_wait(a, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(a, parity)) {
    if (clock64() - t0 > (1ll << 34)) {
      printf("b2: mbarrier wait timeout (smem 0x%x parity %u) block %d thread %d\n", a, parity,
             blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}
B2_DEV void mbar_arrive_expect_tx_u32(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

// ---------------------------------------------------------------- async copies
// K-major operand descriptors for narrow rows: 64-byte (32 bf16) rows with
// 64B swizzle (SBO = 8 rows x 64 B) and 32-byte (16 bf16) rows with 32B swizzle
B2_DEV uint64_t smem_desc_sw64_k(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;   // SWIZZLE_64B
  return d;
}
B2_DEV uint64_t smem_desc_sw32_k(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;   // SWIZZLE_32B
  return d;
}

B2_DEV void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
B2_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// im2col-mode TMA: `pixelsPerColumn` output positions starting at (n, h, w)
// (lower-corner-adjusted input coordinates), channels [c, c + channelsPerPixel),
// each shifted by the filter offset (off_w, off_h); OOB -> zero fill.
B2_DEV void tma_load_im2col_4d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c, int w,
                               int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(off_w), "h"(off_h)
      : "memory");
}
B2_DEV void tma_load_4d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                        int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
B2_DEV void tma_store_3d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
B2_DEV void tma_store_4d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2,
                         int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
B2_DEV void tma_store_2d(const CUtensorMap* map, const void* smem_src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
B2_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> B2_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N> B2_DEV void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
B2_DEV void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 16-byte cp.async with zero fill when src_bytes == 0
B2_DEV void cp_async_16(uint32_t smem_dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}
// arrive on `bar` once all prior cp.async of this thread have landed; the
// arrival counts toward the barrier's expected count (.noinc)
B2_DEV void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
B2_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> B2_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- programmatic dependent launch
// tcgen05 kernels are launched with programmatic stream serialisation: the
// next kernel's CTAs are scheduled (barrier init, TMEM alloc, tensor-map
// prefetch) while this one drains, and block in pdl_wait() until it has
// completed and its writes are visible.  Both are no-ops without the launch
// attribute.
B2_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
B2_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();   // runtime switch (B2_PDL, default on)

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}

// ---------------------------------------------------------------- warp-uniform helpers
// ptxas keeps TMEM addresses and UMMA descriptors in uniform registers only
// when it can prove them warp-uniform; values derived from threadIdx or from
// a shared-memory load are not, and every tcgen05.mma / tcgen05.ld then gets a
// per-instruction ELECT + R2UR.BROADCAST waterfall (~100+ cycles per MMA,
// measured: a 128x64x16 MMA stream ran at 23% tensor-pipe).  So the issuing
// warp runs converged, derives everything from shfl-broadcast values, and
// issues from one elected lane.
B2_DEV int warp_index_uniform() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }
B2_DEV uint32_t uniform_u32(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }
// elect.sync names the full warp: the warp is reconverged first (lanes leave
// an mbarrier poll loop in different iterations, and an elect.sync over a split
// warp elects one lane per fragment — two producers arriving on one barrier).
B2_DEV bool elect_one() {
  __syncwarp();
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- tcgen05 / TMEM
B2_DEV void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
B2_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
B2_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
B2_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate)
B2_DEV void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::tf32 (fp32 storage, tf32 math, fp32 accumulate); K per instruction = 8
B2_DEV void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// all prior tcgen05 async ops of this thread arrive on `bar` when complete
B2_DEV void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
B2_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
B2_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
B2_DEV void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// K-major operand tile in the canonical 128-byte-swizzled layout: rows of
// 128 B (64 bf16 / 32 fp32), 8-row atoms of 1024 B (SBO), base 1024-B aligned.
B2_DEV uint64_t smem_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)(16 >> 4) << 16;     // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

// K-major operand in the non-swizzled ("interleave") canonical layout: core
// matrices of 8 rows x 16 B stored contiguously (128 B); `lbo` = byte stride
// between core matrices along K, `sbo` = byte stride between 8-row groups.
B2_DEV uint64_t smem_desc_kmajor_noswizzle(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;   // layout type 0 = SWIZZLE_NONE
}

// ---------------------------------------------------------------- CTA pairs (cta_group::2)
B2_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
B2_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of this CTA's variable `p` as seen in CTA `rank`
B2_DEV uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// Relaxed: the only cross-CTA arrivals are accumulator releases issued after
// tcgen05.wait::ld, so there is nothing for a release to order — and
// .release.cluster compiles to MEMBAR.ALL.GPU + ERRBAR before the arrive
// (ncu: ~7% of the stall samples of the BERT FFN-up GEMM, every tile, every
// epilogue warp of the peer CTA).
B2_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA loads whose completion is signalled on the pair leader's mbarrier
B2_DEV void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
B2_DEV void tma_load_4d_pair(void* smem_dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                             int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
B2_DEV void tma_load_im2col_4d_pair(void* smem_dst, const CUtensorMap* map, uint32_t bar_cluster,
                                    int c, int w, int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(off_w), "h"(off_h)
      : "memory");
}
B2_DEV void tma_load_2d_u32(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
B2_DEV void tma_load_4d_u32(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
B2_DEV void tma_load_im2col_4d_u32(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c,
                                   int w, int h, int n, uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(off_w), "h"(off_h)
      : "memory");
}
B2_DEV void tma_load_2d_pair_u32(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster,
                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
B2_DEV void tma_load_im2col_4d_pair_u32(uint32_t dst, const CUtensorMap* map,
                                        uint32_t bar_cluster, int c, int w, int h, int n,
                                        uint16_t off_w, uint16_t off_h) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(off_w), "h"(off_h)
      : "memory");
}
B2_DEV void tmem_alloc_pair(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
B2_DEV void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// D[tmem, both CTAs] (+)= A[smem, M = 256 across the pair] * B[smem, N split]^T
B2_DEV void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive (once each) on the mbarrier at this offset in both CTAs of the pair
B2_DEV void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// instruction descriptor: fp32 accumulate, A/B format fmt (1 = bf16, 2 = tf32),
// both K-major, shape M x N
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, uint32_t fmt) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
