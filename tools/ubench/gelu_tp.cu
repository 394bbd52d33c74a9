// Dev microbenchmark (not product): epilogue GELU throughput per SM on sm_100a, for the variants
// the GEMM1 epilogue could use.  Each thread evaluates (h, gp) for 32 values per iteration, like
// one 32-column TMEM chunk.  Prints elements / SM / clock.
#include <cstdio>
#include "../../paper_2112_14397_b200/csrc/common.cuh"
using namespace moe;

// FMA-pipe reciprocal for x in [1, 2^24): magic seed + 3 Newton steps (packed)
__device__ __forceinline__ f32x2 rcp_nr2(f32x2 X) {
  float x0, x1; f2_split(X, x0, x1);
  f32x2 R = f2(__uint_as_float(0x7EF311C3u - __float_as_uint(x0)), __uint_as_float(0x7EF311C3u - __float_as_uint(x1)));
  const f32x2 NX = mul2(X, f2(-1.f));
  #pragma unroll
  for (int i = 0; i < 3; ++i) { f32x2 E = fma2(NX, R, f2(1.f)); R = fma2(R, E, R); }
  return R;
}
// FMA-pipe 2^s for s <= 0 (clamped at -126): round-to-nearest split + degree-6 polynomial
__device__ __forceinline__ f32x2 exp2_poly2(f32x2 S) {
  float s0, s1; f2_split(S, s0, s1);
  s0 = fmaxf(s0, -126.f); s1 = fmaxf(s1, -126.f);
  const f32x2 Sc = f2(s0, s1);
  const f32x2 J = add2(Sc, f2(12582912.f));           // 1.5*2^23: round to nearest integer
  const f32x2 Jr = add2(J, f2(-12582912.f));
  const f32x2 F = add2(Sc, mul2(Jr, f2(-1.f)));        // f in [-0.5, 0.5]
  f32x2 P = fma2(f2(1.535336188e-4f), F, f2(1.339887440e-3f));
  P = fma2(P, F, f2(9.618437357e-3f));
  P = fma2(P, F, f2(5.550332471e-2f));
  P = fma2(P, F, f2(2.402264791e-1f));
  P = fma2(P, F, f2(6.931472028e-1f));
  P = fma2(P, F, f2(1.f));
  float p0, p1, j0, j1; f2_split(P, p0, p1); f2_split(J, j0, j1);
  return f2(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(j0) << 23)),
            __uint_as_float(__float_as_uint(p1) + (__float_as_uint(j1) << 23)));
}

// V = 5: X = 1 + k|a| as ONE FFMA2 on a sign-carrying constant (LOP3 puts a's sign on k);
// V = 6: additionally (1 - NS)/2 from the sign bit on the ALU (SHF + LOP3) instead of an FFMA2
__device__ __forceinline__ uint32_t sign_or(uint32_t a, uint32_t k) {
  uint32_t d;   // (a & 0x80000000) | k
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(0x80000000u), "r"(k));
  return d;
}
__device__ __forceinline__ uint32_t one_if_nonneg(uint32_t a) {
  return (uint32_t)(~((int32_t)a >> 31)) & 0x3f800000u;   // a >= 0 (sign clear) -> 1.0f, else 0
}
template <int V>
__device__ __forceinline__ void gelu2_lean(f32x2 A, f32x2& H, f32x2& G) {
  constexpr float kS2P = 2.5066282746310002f;
  constexpr float kk = 0.3275911f * 0.70710678118654752f;
  float a0, a1;
  f2_split(A, a0, a1);
  const uint32_t ua0 = __float_as_uint(a0), ua1 = __float_as_uint(a1);
  const f32x2 SGK = f2(__uint_as_float(sign_or(ua0, __float_as_uint(kk))), __uint_as_float(sign_or(ua1, __float_as_uint(kk))));
  const f32x2 NS = f2(__uint_as_float(neg_sign_one(ua0, 0x3f800000u)), __uint_as_float(neg_sign_one(ua1, 0x3f800000u)));
  const f32x2 X = fma2(A, SGK, f2(1.0f));
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
  const f32x2 E = f2(ex2_approx(s0), ex2_approx(s1));
  const f32x2 Q = mul2(P, E);
  f32x2 PH;
  if (V == 7) {            // Phi = 0.5 + NS (Q - 0.5): one FFMA2 fewer, absolute (not relative) tail accuracy
    PH = fma2(NS, fma2(P, E, f2(-0.5f)), f2(0.5f));
  } else {
    f32x2 HS;
    if (V == 6) HS = f2(__uint_as_float(one_if_nonneg(ua0)), __uint_as_float(one_if_nonneg(ua1)));
    else HS = fma2(NS, f2(-0.5f), f2(0.5f));
    PH = fma2(NS, Q, HS);
  }
  H = mul2(A, PH);
  G = fma2(A, E, PH);
}

template <int V>
__device__ __forceinline__ void gelu2(f32x2 A, f32x2& H, f32x2& G) {
  if (V == 5 || V == 6 || V == 7) {
    gelu2_lean<V>(A, H, G);
  } else if (V == 0) {
    float a0, a1, h0, h1, g0, g1; f2_split(A, a0, a1);
    gelu_and_prime_fast(a0, h0, g0); gelu_and_prime_fast(a1, h1, g1);
    H = f2(h0, h1); G = f2(g0, g1);
  } else if (V == 1) {
    gelu_and_prime_x2(A, H, G);
  } else {
    float a0, a1; f2_split(A, a0, a1);
    const uint32_t ns0 = (~__float_as_uint(a0) & 0x80000000u) | 0x3f800000u;
    const uint32_t ns1 = (~__float_as_uint(a1) & 0x80000000u) | 0x3f800000u;
    const f32x2 NS = f2(__uint_as_float(ns0), __uint_as_float(ns1));
    const f32x2 X = fma2(mul2(A, NS), f2(-0.3275911f * 0.70710678118654752f), f2(1.0f));
    f32x2 T;
    if (V == 2 || V == 4) T = rcp_nr2(X);
    else { float x0, x1; f2_split(X, x0, x1); T = f2(rcp_approx(x0), rcp_approx(x1)); }
    f32x2 P = fma2(f2(0.5f * 1.061405429f), T, f2(0.5f * -1.453152027f));
    P = fma2(P, T, f2(0.5f * 1.421413741f));
    P = fma2(P, T, f2(0.5f * -0.284496736f));
    P = fma2(P, T, f2(0.5f * 0.254829592f));
    P = mul2(T, P);
    const f32x2 S = mul2(A, mul2(A, f2(-0.5f * 1.4426950408889634f)));
    f32x2 E;
    if (V == 3 || V == 4) E = exp2_poly2(S);
    else { float s0, s1; f2_split(S, s0, s1); E = f2(ex2_approx(s0), ex2_approx(s1)); }
    const f32x2 Q = mul2(P, E);
    const f32x2 PH = fma2(NS, Q, fma2(NS, f2(-0.5f), f2(0.5f)));
    H = mul2(A, PH);
    G = fma2(mul2(A, f2(0.39894228040143268f)), E, PH);
  }
}

template <int V>
__global__ void __launch_bounds__(384) k(float* out, long long* clk, int iters, float seed) {
  f32x2 v[16], acc = f2(0.f);
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = f2(seed * (threadIdx.x + j) * 1e-3f - 2.f, seed * (threadIdx.x - j) * 1e-3f + 1.f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      f32x2 h, g;
      gelu2<V>(v[j], h, g);
      acc = add2(acc, add2(h, g));
      v[j] = add2(v[j], f2(1e-3f));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float a0, a1; f2_split(acc, a0, a1);
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// raw pipe throughputs
template <int W>
__global__ void __launch_bounds__(384) raw(float* out, long long* clk, int iters) {
  float x[8]; f32x2 y[8];
  for (int j = 0; j < 8; ++j) { x[j] = 1.f + threadIdx.x * 1e-4f + j; y[j] = f2(x[j], x[j] + 1.f); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (W == 0) x[j] = ex2_approx(x[j] * -0.001f);
      if (W == 1) x[j] = rcp_approx(x[j]);
      if (W == 2) x[j] = fmaf(x[j], 0.9999f, 1e-4f);
      if (W == 3) y[j] = fma2(y[j], f2(0.9999f), f2(1e-4f));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) { float a, b; f2_split(y[j], a, b); s += x[j] + a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int V>
__global__ void acc_k(double* err, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n / 2) return;
  float a0 = -10.f + 20.f * (2 * i) / n, a1 = -10.f + 20.f * (2 * i + 1) / n;
  f32x2 H, G; gelu2<V>(f2(a0, a1), H, G);
  float h[2], g[2]; f2_split(H, h[0], h[1]); f2_split(G, g[0], g[1]);
  float a[2] = {a0, a1};
  for (int q = 0; q < 2; ++q) {
    double ad = a[q], ph = 0.5 * erfc(-ad / sqrt(2.0)), hr = ad * ph, gr = ph + ad * exp(-0.5 * ad * ad) / sqrt(2 * M_PI);
    atomicMax((unsigned long long*)&err[0], __double_as_longlong(fabs(h[q] - hr)));
    atomicMax((unsigned long long*)&err[1], __double_as_longlong(fabs(g[q] - gr)));
  }
}

int main() {
  {
    double* e; cudaMalloc(&e, 16); double he[2]; const int n = 1 << 22;
#define ACC(V) cudaMemset(e, 0, 16); acc_k<V><<<n / 512, 256>>>(e, n); cudaMemcpy(he, e, 16, cudaMemcpyDeviceToHost); \
    printf("variant %d: max|h err| %.3e  max|gp err| %.3e\n", V, he[0], he[1]);
    ACC(0) ACC(1) ACC(2) ACC(3) ACC(4) ACC(5) ACC(6) ACC(7)
  }
  float* out; long long* clk; cudaMalloc(&out, 148 * 384 * 4); cudaMalloc(&clk, 148 * 8);
  long long h[148];
  const int iters = 2000;
  auto report = [&](const char* name, double per_thread_iter) {
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("%-28s %8.2f per SM per clock\n", name, 384.0 * iters * per_thread_iter / c);
  };
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<148, 384>>>(out, clk, iters, 1.f); report("gelu scalar (elem)", 32);
    k<1><<<148, 384>>>(out, clk, iters, 1.f); report("gelu x2 MUFU (elem)", 32);
    k<2><<<148, 384>>>(out, clk, iters, 1.f); report("gelu x2 NR-rcp (elem)", 32);
    k<3><<<148, 384>>>(out, clk, iters, 1.f); report("gelu x2 poly-exp2 (elem)", 32);
    k<4><<<148, 384>>>(out, clk, iters, 1.f); report("gelu x2 no MUFU (elem)", 32);
    k<5><<<148, 384>>>(out, clk, iters, 1.f); report("gelu x2 sign-k X (elem)", 32);
    k<6><<<148, 384>>>(out, clk, iters, 1.f); report("gelu x2 sign-k X + ALU HS (elem)", 32);
    k<7><<<148, 384>>>(out, clk, iters, 1.f); report("gelu x2 sign-k X + Q-0.5 (elem)", 32);
    raw<0><<<148, 384>>>(out, clk, iters); report("MUFU.EX2 (+FMUL)", 8);
    raw<1><<<148, 384>>>(out, clk, iters); report("MUFU.RCP", 8);
    raw<2><<<148, 384>>>(out, clk, iters); report("FFMA", 8);
    raw<3><<<148, 384>>>(out, clk, iters); report("FFMA2 (lanes)", 16);
  }
  return 0;
}
