// common.cuh -- shared device helpers for the DTS-Gate MoE kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace moe {

constexpr int kRowAlign = 128;          // MOE_ROW_ALIGN
constexpr int kWarp = 32;

// device error flag bits (workspace word 0)
constexpr int kFlagNonFinite = 1;
constexpr int kFlagCapacity = 2;
constexpr int kFlagArrival = 4;    // overlap mode: an expert's rows did not all arrive in time

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(bf16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f32<bf16>(float v) { return __float2bfloat16_rn(v); }

// 16-byte vector of T: 4 floats or 8 bf16
template <typename T> struct Vec16;
template <> struct Vec16<float> { static constexpr int N = 4; };
template <> struct Vec16<bf16> { static constexpr int N = 8; };

__device__ __forceinline__ void unpack16(const uint4& v, float* out, float) {
  out[0] = __uint_as_float(v.x); out[1] = __uint_as_float(v.y);
  out[2] = __uint_as_float(v.z); out[3] = __uint_as_float(v.w);
}
__device__ __forceinline__ void unpack16(const uint4& v, float* out, bf16) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = __uint_as_float(w[i] << 16);
    out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
__device__ __forceinline__ uint4 pack16(const float* in, float) {
  return make_uint4(__float_as_uint(in[0]), __float_as_uint(in[1]), __float_as_uint(in[2]),
                    __float_as_uint(in[3]));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}
__device__ __forceinline__ uint4 pack16(const float* in, bf16) {
  return make_uint4(pack_bf16x2(in[0], in[1]), pack_bf16x2(in[2], in[3]), pack_bf16x2(in[4], in[5]),
                    pack_bf16x2(in[6], in[7]));
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_nc_f4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  return *reinterpret_cast<const uint4*>(p);
}
__device__ __forceinline__ void st_v4(void* p, const uint4& v) { *reinterpret_cast<uint4*>(p) = v; }

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// GELU, erf form (Eq. 3 with GeLU per P:472; reading R8)
__device__ __forceinline__ float gelu_f(float a) { return 0.5f * a * (1.0f + erff(a * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_prime_f(float a) {
  return 0.5f * (1.0f + erff(a * 0.70710678118654752f)) +
         a * 0.39894228040143268f * __expf(-0.5f * a * a);
}

// Epilogue-grade Phi(a) = (1 + erf(a/sqrt2))/2 from Abramowitz & Stegun 7.1.26
// (|erf error| <= 1.5e-7, far below the bf16 rounding of a and h): for x = |a|/sqrt2,
// erfc(x) = t*(a1 + t*(a2 + ... a5)) * exp(-x^2), t = 1/(1 + p x).  The 1/2 of Phi is folded
// into the coefficients; exp(-x^2) = exp(-a^2/2) is returned for phi(a) = exp(-a^2/2)/sqrt(2 pi).
// One MUFU.RCP + one MUFU.EX2 per element.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float phi_cdf_as(float a, float& e) {
  const float t = rcp_approx(fmaf(0.3275911f * 0.70710678118654752f, fabsf(a), 1.0f));
  const float poly = t * fmaf(fmaf(fmaf(fmaf(0.5f * 1.061405429f, t, 0.5f * -1.453152027f), t, 0.5f * 1.421413741f), t,
                                   0.5f * -0.284496736f),
                              t, 0.5f * 0.254829592f);
  e = ex2_approx(a * (a * (-0.5f * 1.4426950408889634f)));   // exp(-a^2/2)
  const float q = poly * e;                                  // erfc(|a|/sqrt2) / 2 = Phi(-|a|)
  return a >= 0.0f ? 1.0f - q : q;
}
__device__ __forceinline__ float gelu_fast(float a) {
  float e;
  return a * phi_cdf_as(a, e);
}
// GELU'(a) = Phi(a) + a phi(a)
__device__ __forceinline__ float gelu_prime_fast(float a) {
  float e;
  const float ph = phi_cdf_as(a, e);
  return fmaf(a * 0.39894228040143268f, e, ph);
}
// Both at once from one Phi(a) / exp(-a^2/2): h = GELU(a), gp = GELU'(a).
__device__ __forceinline__ void gelu_and_prime_fast(float a, float& h, float& gp) {
  float e;
  const float ph = phi_cdf_as(a, e);
  h = a * ph;
  gp = fmaf(a * 0.39894228040143268f, e, ph);
}

// ---- packed fp32x2 (sm_100a FFMA2/FMUL2/FADD2): two lanes of fp32 per instruction, each lane
// rounded exactly like its scalar counterpart, so results are bit-identical to the scalar code.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f32x2 f2(float v) { return f2(v, v); }
__device__ __forceinline__ void f2_split(f32x2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// bf16x2 word -> fp32 pair (low half = first element)
__device__ __forceinline__ f32x2 bf16x2_to_f2(uint32_t w) {
  return f2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
__device__ __forceinline__ uint32_t f2_to_bf16x2(f32x2 v) {
  float lo, hi;
  f2_split(v, lo, hi);
  return pack_bf16x2(lo, hi);
}

// gelu_and_prime_fast on two elements with the packed pipe (same approximation; the constant
// folding below changes the last-bit rounding, not the |erf error| <= 1.5e-7 bound): with
// ns = -sign(a) (as +-1), -|a| = a*ns, t = rcp(1 + k|a|) = rcp(fma(-|a|, -k, 1)),
// Phi = fma(ns, q, (1 - ns)/2), i.e. 1 - q for a >= 0 and q for a < 0 (the scalar select).
// Instruction-lean form (GEMM1 epilogue): the sign word ns = (~a & 0x80000000) | 1.0f is one
// LOP3 per element (1.0f held in a register), and 1/sqrt(2 pi) is folded into the exponent
// (E' = exp(-a^2/2) / sqrt(2 pi) = ex2(-a^2 log2(e)/2 - log2(2 pi)/2) = phi(a)) and, inversely,
// into the erfc polynomial, so q = P' E' is unchanged and GELU'(a) = Phi + a phi = fma(a, E', Phi).
__device__ __forceinline__ uint32_t neg_sign_one(uint32_t a, uint32_t one) {
  uint32_t d;   // (~a & 0x80000000) | one   (LUT 0xAE: f(a=F0, b=CC, c=AA) = (~a & b) | c)
  asm("lop3.b32 %0, %1, %2, %3, 0xAE;" : "=r"(d) : "r"(a), "n"(0x80000000u), "r"(one));
  return d;
}
__device__ __forceinline__ void gelu_and_prime_x2(f32x2 A, f32x2& H, f32x2& G, bool want_g = true) {
  constexpr float kS2P = 2.5066282746310002f;   // sqrt(2 pi)
  float a0, a1;
  f2_split(A, a0, a1);
  const uint32_t one = 0x3f800000u;
  const f32x2 NS = f2(__uint_as_float(neg_sign_one(__float_as_uint(a0), one)),
                      __uint_as_float(neg_sign_one(__float_as_uint(a1), one)));
  const f32x2 X = fma2(mul2(A, NS), f2(-0.3275911f * 0.70710678118654752f), f2(1.0f));
  float x0, x1;
  f2_split(X, x0, x1);
  const f32x2 T = f2(rcp_approx(x0), rcp_approx(x1));
  f32x2 P = fma2(f2(0.5f * kS2P * 1.061405429f), T, f2(0.5f * kS2P * -1.453152027f));
  P = fma2(P, T, f2(0.5f * kS2P * 1.421413741f));
  P = fma2(P, T, f2(0.5f * kS2P * -0.284496736f));
  P = fma2(P, T, f2(0.5f * kS2P * 0.254829592f));
  P = mul2(T, P);
  const f32x2 S = fma2(A, mul2(A, f2(-0.5f * 1.4426950408889634f)), f2(-1.3257480647361595f));
  float s0, s1;
  f2_split(S, s0, s1);
  const f32x2 E = f2(ex2_approx(s0), ex2_approx(s1));   // phi(a)
  const f32x2 Q = mul2(P, E);                            // Phi(-|a|)
  const f32x2 PH = fma2(NS, Q, fma2(NS, f2(-0.5f), f2(0.5f)));
  H = mul2(A, PH);
  if (want_g) G = fma2(A, E, PH);
}

}  // namespace moe
