// gate_token.cuh -- steps 2-3 of the DTS gate for one token, executed by one warp
// (lanes = experts): Gumbel noise, tau-softmax, threshold / guard / top-1 decision, fp64
// refinement of near-boundary tokens, band count.  Shared by the SIMT and tcgen05 gates.
#pragma once
#include "common.cuh"

namespace moe {
namespace {

constexpr float kRefine = 5e-5f;
constexpr float kBand = 1e-6f;
constexpr int kMaxEPL = 4;          // experts per lane (E <= 128)

__device__ __forceinline__ void warp_argmax(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
  }
}
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
  }
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_maxd(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Second largest value given the argmax index (for the top-2 gap).
__device__ __forceinline__ float warp_second(const float* p, int E, int lane, int am) {
  float s = -1.f;
#pragma unroll
  for (int i = 0; i < kMaxEPL; ++i) {
    int e = lane + 32 * i;
    if (e < E && e != am) s = fmaxf(s, p[i]);
  }
  return warp_max(s);
}

// Steps 2-3 for one token, executed by one warp.  L points at the token's E fp32 logits.
template <typename T>
__device__ __forceinline__ void gate_token(const float* L, int t, const T* __restrict__ x, const T* __restrict__ Wg,
                                           const float* __restrict__ u, int d, int E, float tau, float thr, int top1,
                                           float* __restrict__ probs, int* __restrict__ slot, int* s_cnt, int* s_band,
                                           int* __restrict__ flags, int lane) {
  float z[kMaxEPL], p[kMaxEPL];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < kMaxEPL; ++i) {
    int e = lane + 32 * i;
    z[i] = -INFINITY;
    if (e < E) {
      float Lv = L[e];
      if (!isfinite(Lv)) bad = true;
      float zeta = u ? -logf(-logf(u[(long long)t * E + e])) : 0.f;
      z[i] = (Lv + zeta) / tau;
    }
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0 && atomicOr(&flags[0], kFlagNonFinite) == 0) flags[1] = t;
  }
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < kMaxEPL; ++i) mx = fmaxf(mx, z[i]);
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxEPL; ++i) {
    p[i] = (lane + 32 * i < E) ? expf(z[i] - mx) : 0.f;
    sum += p[i];
  }
  sum = warp_sum(sum);
  const float inv = 1.0f / sum;
  bool any_pass = false, near = false;
  float pmax = -1.f;
  int am = 0x7fffffff;
#pragma unroll
  for (int i = 0; i < kMaxEPL; ++i) {
    int e = lane + 32 * i;
    if (e < E) {
      p[i] = p[i] * inv;
      if (p[i] > thr) any_pass = true;
      if (fabsf(p[i] - thr) < kRefine) near = true;
      if (p[i] > pmax) { pmax = p[i]; am = e; }
    }
  }
  warp_argmax(pmax, am);
  any_pass = __any_sync(0xffffffffu, any_pass);
  bool argmax_decided = top1 || !any_pass;
  near = __any_sync(0xffffffffu, near) && !top1;
  if (argmax_decided) {
    float second = warp_second(p, E, lane, am);
    if (pmax - second < kRefine) near = true;
  }
  if (near) {
    // ---- fp64 refinement: recompute logits, noise and softmax exactly from the inputs
    double z64[kMaxEPL];
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i) {
      int e = lane + 32 * i;
      z64[i] = -INFINITY;
      if (e < E) {
        double acc = 0.0;
        const T* xr = x + (long long)t * d;
        for (int k = 0; k < d; ++k) acc = fma((double)to_f32(xr[k]), (double)to_f32(Wg[(long long)k * E + e]), acc);
        double zeta = u ? -log(-log((double)u[(long long)t * E + e])) : 0.0;
        z64[i] = (acc + zeta) / (double)tau;
      }
    }
    double mx64 = -INFINITY;
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i) mx64 = fmax(mx64, z64[i]);
    mx64 = warp_maxd(mx64);
    double s64 = 0.0, p64[kMaxEPL];
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i) {
      p64[i] = (lane + 32 * i < E) ? exp(z64[i] - mx64) : 0.0;
      s64 += p64[i];
    }
    s64 = warp_sum(s64);
    double best = -1.0;
    int bi = 0x7fffffff;
    any_pass = false;
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i) {
      int e = lane + 32 * i;
      if (e < E) {
        p64[i] /= s64;
        p[i] = (float)p64[i];
        if (p[i] > thr) any_pass = true;
        if (p64[i] > best) { best = p64[i]; bi = e; }
      }
    }
    warp_argmax(best, bi);
    am = bi;
    pmax = (float)best;
    any_pass = __any_sync(0xffffffffu, any_pass);
    argmax_decided = top1 || !any_pass;
  }
  // ---- decision + band
  bool in_band = false;
  if (!argmax_decided) {
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i)
      if (lane + 32 * i < E && fabsf(p[i] - thr) < kBand) in_band = true;
    in_band = __any_sync(0xffffffffu, in_band);
  } else {
    float second = warp_second(p, E, lane, am);
    in_band = (pmax - second) < kBand;
  }
#pragma unroll
  for (int i = 0; i < kMaxEPL; ++i) {
    int e = lane + 32 * i;
    if (e < E) {
      bool sel = argmax_decided ? (e == am) : (p[i] > thr);
      probs[(long long)t * E + e] = p[i];
      slot[(long long)t * E + e] = sel ? 0 : -1;
      if (sel) atomicAdd(&s_cnt[e], 1);
    }
  }
  if (lane == 0 && in_band) atomicAdd(s_band, 1);
}



// fp64 decision for one token deferred by the thread-per-token fast path (near the
// threshold or an argmax tie), computed by a whole NT-thread block.  The fp64 logits are a
// latency problem (one token: d * E products), so W_g is staged through shared memory in
// chunks of up to 32 KB, each chunk's loads all issued before any is used (one memory
// round trip per chunk, not one per k step); thread (e, sl) then accumulates expert e over
// the k = sl (mod nsl) rows of the chunk (the next chunk's loads in flight meanwhile), the nsl
// partials are added in fixed order; noise (computed during the first loads), tau and the
// exponentials run one expert per thread, and warp 0 takes max / sum / decision in fp64,
// writes probs / slot and counts with global integer atomics.
constexpr int kRefineWBytes = 32768;
constexpr int kRefineKC = 1024;
struct RefineSmem {
  uint4 w[kRefineWBytes / 16];     // W_g rows [k0, k0 + KC) of this chunk, raw element type
  double x[kRefineKC];             // x[k0 .. k0 + KC), converted once per chunk
  double red[1024];                // per-thread partial logits (NT <= 1024)
};
static_assert(sizeof(RefineSmem) <= 48 * 1024, "static shared memory");

// Exact bf16 -> fp64 with integer ops (the F2F.F64.F32 conversion runs on a slow pipe and was
// two per product): a normal value rebiases its exponent (127 -> 1023) and moves its 7
// mantissa bits to the top of the 52; zero, subnormals, inf and NaN take the conversion.
__device__ __forceinline__ double to_f64(bf16 v) {
  const uint32_t b = __bfloat16_as_ushort(v);
  const uint32_t em = b & 0x7fffu;
  if (em - 0x0080u < 0x7f00u)
    return __hiloint2double((int)(((b & 0x8000u) << 16) | ((em << 13) + (896u << 20))), 0);
  return (double)__uint_as_float(b << 16);
}
__device__ __forceinline__ double to_f64(float v) { return (double)v; }

template <typename T, int NT = 256>
__device__ __forceinline__ void gate_token_refine_block(int t, const T* __restrict__ x, const T* __restrict__ Wg,
                                                        const float* __restrict__ u, int d, int E, float tau,
                                                        float thr, int top1, float* __restrict__ probs,
                                                        int* __restrict__ slot, int* __restrict__ counts,
                                                        int* __restrict__ blk_cnt, int nblk, int blk_tokens,
                                                        int* __restrict__ near_band, RefineSmem& sm) {
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const T* xr = x + (long long)t * d;
  static_assert(NT <= 1024 && NT % 32 == 0, "block size");
  const int nsl = NT / E;                         // E <= 128: >= 2 k slices
  const int e_me = tid % E, sl = tid / E;
  const bool worker = sl < nsl;
  int KC = kRefineWBytes / (E * (int)sizeof(T));
  if (KC > kRefineKC) KC = kRefineKC;
  const T* ws = reinterpret_cast<const T*>(sm.w);
  const bool vec = ((E * sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(Wg) & 15) == 0);
  // the token's Gumbel noise in fp64 (two dependent logs), one expert per thread, computed
  // while the first W_g chunk is in flight
  double zeta_me = 0.0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  constexpr int WJ = (kRefineWBytes / 16 + NT - 1) / NT;
  constexpr int XJ = (kRefineKC + NT - 1) / NT;
  uint4 wr[WJ];                                   // vec path: the next chunk's W_g, prefetched
  T xv[XJ];                                       // the next chunk's x
  auto load_chunk = [&](int k0) {
    const int kc = min(KC, d - k0);
    if (vec) {
      const uint4* src = reinterpret_cast<const uint4*>(Wg + (long long)k0 * E);
      const int n16 = (int)((long long)kc * E * sizeof(T) / 16);   // <= 2048
#pragma unroll
      for (int j = 0; j < WJ; ++j)
        if (tid + NT * j < n16) wr[j] = __ldg(src + tid + NT * j);
    }
#pragma unroll
    for (int j = 0; j < XJ; ++j)
      if (tid + NT * j < kc) xv[j] = xr[k0 + tid + NT * j];
  };
  load_chunk(0);
  if (tid < E && u) zeta_me = -log(-log((double)u[(long long)t * E + tid]));
  for (int k0 = 0; k0 < d; k0 += KC) {
    const int kc = min(KC, d - k0);
    const long long n = (long long)kc * E;         // elements of this chunk
    if (vec) {
      const int n16 = (int)(n * sizeof(T) / 16);
#pragma unroll
      for (int j = 0; j < WJ; ++j)
        if (tid + NT * j < n16) sm.w[tid + NT * j] = wr[j];
    } else {
      T* wd = reinterpret_cast<T*>(sm.w);
      for (int b = 0; b < n; b += NT * 8) {
        T r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (b + tid + NT * j < n) r[j] = Wg[(long long)k0 * E + b + tid + NT * j];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (b + tid + NT * j < n) wd[b + tid + NT * j] = r[j];
      }
    }
#pragma unroll
    for (int j = 0; j < XJ; ++j)
      if (tid + NT * j < kc) sm.x[tid + NT * j] = to_f64(xv[j]);
    __syncthreads();
    if (k0 + KC < d) load_chunk(k0 + KC);          // in flight during this chunk's products
    if (worker) {   // four independent fp64 chains in registers
      const T* wc = ws + e_me;
      int k = sl;
      for (; k + 3 * nsl < kc; k += 4 * nsl) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          acc[j] = fma(sm.x[k + j * nsl], to_f64(wc[(k + j * nsl) * E]), acc[j]);
      }
      for (; k < kc; k += nsl) acc[0] = fma(sm.x[k], to_f64(wc[k * E]), acc[0]);
    }
    __syncthreads();
  }
  sm.red[tid] = worker ? (acc[0] + acc[1]) + (acc[2] + acc[3]) : 0.0;
  __syncthreads();
  // noise and tau, then the softmax exponentials, one expert per thread (the W_g staging area
  // is free now: zs[0..E) = z, then p unnormalised; zs[128] = max z); warp 0 decides
  double* zs = reinterpret_cast<double*>(sm.w);
  if (tid < E) {
    double a = 0.0;
    for (int q = 0; q < nsl; ++q) a += sm.red[q * E + tid];
    zs[tid] = (a + zeta_me) / (double)tau;
  }
  __syncthreads();
  if (warp == 0) {
    double mx64 = -INFINITY;
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i)
      if (lane + 32 * i < E) mx64 = fmax(mx64, zs[lane + 32 * i]);
    mx64 = warp_maxd(mx64);
    if (lane == 0) zs[128] = mx64;
  }
  __syncthreads();
  if (tid < E) zs[tid] = exp(zs[tid] - zs[128]);
  __syncthreads();
  if (warp == 0) {
    double s64 = 0.0, p64[kMaxEPL];
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i) {
      p64[i] = (lane + 32 * i < E) ? zs[lane + 32 * i] : 0.0;
      s64 += p64[i];
    }
    s64 = warp_sum(s64);
    float p[kMaxEPL];
    double best = -1.0;
    int am = 0x7fffffff;
    bool any_pass = false;
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i) {
      const int e = lane + 32 * i;
      p[i] = 0.f;
      if (e < E) {
        p64[i] /= s64;
        p[i] = (float)p64[i];
        if (p[i] > thr) any_pass = true;
        if (p64[i] > best) { best = p64[i]; am = e; }
      }
    }
    warp_argmax(best, am);
    any_pass = __any_sync(0xffffffffu, any_pass);
    const bool argmax_decided = top1 || !any_pass;
    const float pmax = (float)best;
    bool in_band = false;
    if (!argmax_decided) {
#pragma unroll
      for (int i = 0; i < kMaxEPL; ++i)
        if (lane + 32 * i < E && fabsf(p[i] - thr) < kBand) in_band = true;
      in_band = __any_sync(0xffffffffu, in_band);
    } else {
      const float second = warp_second(p, E, lane, am);
      in_band = (pmax - second) < kBand;
    }
    const int blk = t / blk_tokens;
#pragma unroll
    for (int i = 0; i < kMaxEPL; ++i) {
      const int e = lane + 32 * i;
      if (e < E) {
        const bool sel = argmax_decided ? (e == am) : (p[i] > thr);
        probs[(long long)t * E + e] = p[i];
        slot[(long long)t * E + e] = sel ? 0 : -1;
        if (sel) {
          atomicAdd(&counts[e], 1);
          atomicAdd(&blk_cnt[(long long)e * nblk + blk], 1);
        }
      }
    }
    if (lane == 0 && in_band) atomicAdd(near_band, 1);
  }
  __syncthreads();
}

}  // namespace
}  // namespace moe
