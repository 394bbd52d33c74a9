// gate.cu -- DTS gate forward (steps 1-3) and backward (B1-3), balance loss (NEXT #1).
//
// Step 1  L = x W_g                                  Eq. 6
// Step 2  p = softmax_E((L + zeta)/tau), zeta = -log(-log u)     Eq. 8, P:330-333 (R1, R2)
// Step 3  m = [p > c] (strict), argmax guard; or top-1           Eq. 9, Alg. 2
//
// Routing precision: logits are accumulated in fp32.
// Any token with an entry |p - c| < kRefine (dense branch), or whose decision is
// argmax-based with a top-2 gap < kRefine, is recomputed entirely in fp64 from the
// same inputs before deciding, so the selection equals the fp64 definition except
// for entries within ~1e-7 of c.
#include "common.cuh"
#include "internal.h"
#include "gate_token.cuh"

namespace moe {

namespace {

// Fused gate: one CTA per kGateBT (128) tokens, 256 threads.
//   Step 1 on CUDA cores: thread = TPT tokens x 4 experts; K in chunks of KC = 32 staged in
//   smem as fp32; chunk partial sums are added with TwoSum (error-free transformation), so
//   the fp32 logits carry ~1 ulp of error instead of the ~sqrt(d) ulp of a plain running
//   sum (the 1e-5 probs tolerance at tau = 0.05..0.1 needs it).
//   Steps 2-3: warp per token on the smem logits (gate_token).
constexpr int kKC = 32;
template <typename T, int TPT, int kGateThreads>   // kGateThreads / 256 k-groups
__global__ void __launch_bounds__(kGateThreads) gate_fused_kernel(
    const T* __restrict__ x, const T* __restrict__ Wg, const float* __restrict__ u, int T_, int d, int E, float tau,
    float thr, int top1, float* __restrict__ probs, int* __restrict__ slot, int* __restrict__ counts,
    int* __restrict__ blk_cnt, int* __restrict__ near_band, int* __restrict__ flags) {
  extern __shared__ float sm[];
  __shared__ int s_cnt[128];
  __shared__ int s_band;
  const int EG = (E + 3) / 4;
  const int Ep = EG * 4;
  float* xs = sm;                          // [kKC][kGateBT + 4]
  float* ws = xs + kKC * (kGateBT + 4);    // [kKC][Ep]
  float* ls = ws + kKC * Ep;               // [kGateBT][E + 1]   logits (sum part)
  float* lc = ls + kGateBT * (E + 1);      // [kGateBT][E + 1]   compensation part
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int t0 = blockIdx.x * kGateBT;
  for (int i = tid; i < E; i += kGateThreads) s_cnt[i] = 0;
  if (tid == 0) s_band = 0;
  // thread = (k-group ks, token group tg, expert group eg): ks owns k-steps [ks*KG, ks*KG + KG) of each chunk
  constexpr int KS = kGateThreads / 256, KG = kKC / KS;
  const int ks = tid / 256, tl = tid % 256;
  const int eg = tl % EG, tg = tl / EG;
  const bool active = tg * TPT < kGateBT;
  float sum[TPT][4], comp[TPT][4];
#pragma unroll
  for (int i = 0; i < TPT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) sum[i][j] = comp[i][j] = 0.f;
  constexpr int V = Vec16<T>::N;
  for (int k0 = 0; k0 < d; k0 += kKC) {
    // x chunk: kGateBT tokens x kKC, 16-byte vectors
    for (int v = tid; v < kGateBT * (kKC / V); v += kGateThreads) {
      const int tok = v / (kKC / V), part = v % (kKC / V);
      const int kk = part * V;
      float f[V];
      if (t0 + tok < T_ && k0 + kk < d) {
        unpack16(ld_nc_v4(x + (long long)(t0 + tok) * d + k0 + kk), f, T());
      } else {
#pragma unroll
        for (int q = 0; q < V; ++q) f[q] = 0.f;
      }
#pragma unroll
      for (int q = 0; q < V; ++q) xs[(kk + q) * (kGateBT + 4) + tok] = f[q];
    }
    for (int i = tid; i < kKC * Ep; i += kGateThreads) {
      const int kk = i / Ep, e = i % Ep;
      ws[i] = (k0 + kk < d && e < E) ? to_f32(Wg[(long long)(k0 + kk) * E + e]) : 0.f;
    }
    __syncthreads();
    if (active) {
      float c[TPT][4];
#pragma unroll
      for (int i = 0; i < TPT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
#pragma unroll
      for (int k2 = 0; k2 < KG; ++k2) {
        const int kk = ks * KG + k2;
        const float4 b = *reinterpret_cast<const float4*>(&ws[kk * Ep + eg * 4]);
        float a[TPT];
#pragma unroll
        for (int i = 0; i < TPT; ++i) a[i] = xs[kk * (kGateBT + 4) + tg * TPT + i];
#pragma unroll
        for (int i = 0; i < TPT; ++i) {
          c[i][0] = fmaf(a[i], b.x, c[i][0]);
          c[i][1] = fmaf(a[i], b.y, c[i][1]);
          c[i][2] = fmaf(a[i], b.z, c[i][2]);
          c[i][3] = fmaf(a[i], b.w, c[i][3]);
        }
      }
#pragma unroll
      for (int i = 0; i < TPT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {   // TwoSum(sum, c) -> (sum, err)
          const float s1 = sum[i][j] + c[i][j];
          const float bp = s1 - sum[i][j];
          const float err = (sum[i][j] - (s1 - bp)) + (c[i][j] - bp);
          sum[i][j] = s1;
          comp[i][j] += err;
        }
    }
    __syncthreads();
  }
  // combine the KS partial (sum, comp) pairs in fixed order ks = 0, 1, ... with TwoSum
  for (int g = 0; g < KS; ++g) {
    if (ks == g && active) {
#pragma unroll
      for (int i = 0; i < TPT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int e = eg * 4 + j;
          if (e >= E) continue;
          const int at = (tg * TPT + i) * (E + 1) + e;
          if (g == 0) {
            ls[at] = sum[i][j];
            lc[at] = comp[i][j];
          } else {
            const float s0 = ls[at];
            const float s1 = s0 + sum[i][j];
            const float bp = s1 - s0;
            const float err = (s0 - (s1 - bp)) + (sum[i][j] - bp);
            ls[at] = s1;
            lc[at] += err + comp[i][j];
          }
        }
    }
    __syncthreads();
  }
  for (int i = tid; i < kGateBT * (E + 1); i += kGateThreads) ls[i] += lc[i];
  __syncthreads();
  for (int i = warp; i < kGateBT; i += kGateThreads / 32) {
    const int t = t0 + i;
    if (t >= T_) break;
    gate_token<T>(&ls[i * (E + 1)], t, x, Wg, u, d, E, tau, thr, top1, probs, slot, s_cnt, &s_band, flags, lane);
  }
  __syncthreads();
  for (int e = tid; e < E; e += kGateThreads) {
    int c = s_cnt[e];
    blk_cnt[(long long)e * gridDim.x + blockIdx.x] = c;   // expert-major [E][nblk]
    if (c) atomicAdd(&counts[e], c);
  }
  if (tid == 0 && s_band) atomicAdd(near_band, s_band);
}

template <typename T, int TPT>
cudaError_t launch_gate_fused(const moe_ctx* c, const void* x, const void* Wg, const float* u, float tau, float thr,
                              int top1, float* probs, int32_t* slot, int32_t* counts, int32_t* near_band,
                              cudaStream_t s) {
  const int Ep = (c->E + 3) / 4 * 4;
  // more k-groups (threads) when the per-thread tile is small; 64/128 registers budget otherwise
  constexpr int kGateThreads = TPT <= 4 ? 1024 : (TPT <= 8 ? 512 : 256);
  const size_t smem = sizeof(float) * (kKC * (kGateBT + 4) + kKC * Ep + 2 * kGateBT * (c->E + 1));
  cudaError_t e = cudaFuncSetAttribute(gate_fused_kernel<T, TPT, kGateThreads>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  gate_fused_kernel<T, TPT, kGateThreads><<<c->nblk, kGateThreads, smem, s>>>((const T*)x, (const T*)Wg, u, c->T, c->d, c->E, tau, thr,
                                                       top1, probs, slot, counts, c->blk_cnt, near_band, c->flags),
      count_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_gate_typed(const moe_ctx* c, const void* x, const void* Wg, const float* u, float tau, float thr,
                              int top1, float* probs, int32_t* slot, int32_t* counts, int32_t* near_band,
                              cudaStream_t s) {
  const int EG = (c->E + 3) / 4;   // TPT >= EG / 2 so that EG * (128 / TPT) <= 256 threads
  if (EG <= 2) return launch_gate_fused<T, 1>(c, x, Wg, u, tau, thr, top1, probs, slot, counts, near_band, s);
  if (EG <= 4) return launch_gate_fused<T, 2>(c, x, Wg, u, tau, thr, top1, probs, slot, counts, near_band, s);
  if (EG <= 8) return launch_gate_fused<T, 4>(c, x, Wg, u, tau, thr, top1, probs, slot, counts, near_band, s);
  if (EG <= 16) return launch_gate_fused<T, 8>(c, x, Wg, u, tau, thr, top1, probs, slot, counts, near_band, s);
  return launch_gate_fused<T, 16>(c, x, Wg, u, tau, thr, top1, probs, slot, counts, near_band, s);
}

// ------------------------------------------------------------------ gate backward
// One warp per token: dp = m dG (+ balance), dz = p (dp - <p,dp>), dlogits = dz / tau.
// PEER (fused peer-memory EP, token side): dG of (t, e) sits at row slot[t,e] of the rank
// owning e, read through its NVLink peer pointer dGp.p[e / El].
template <bool PEER = false>
__global__ void __launch_bounds__(256) gate_bwd_token_kernel(
    const float* __restrict__ dG_row, const int* __restrict__ slot, const float* __restrict__ probs,
    int T_, int E, float tau, float alpha, const int* __restrict__ counts, int count_rows, double bal_scale,
    float* __restrict__ dlogits, bf16* __restrict__ dL2, int Ep, int Kp, int El,
    const __grid_constant__ PeerTable dGp) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t = blockIdx.x * 8 + warp;
  if (t >= T_) return;
  float p[kMaxEPL], dp[kMaxEPL];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxEPL; ++i) {
    int e = lane + 32 * i;
    p[i] = 0.f; dp[i] = 0.f;
    if (e < E) {
      p[i] = probs[(long long)t * E + e];
      int r = slot[(long long)t * E + e];
      dp[i] = r >= 0 ? (PEER ? reinterpret_cast<const float*>(dGp.p[e / El])[r] : dG_row[r]) : 0.f;
      if (alpha > 0.f) {                       // global count of e: the column sum of the count rows
        int ce = 0;
        for (int q = 0; q < count_rows; ++q) ce += counts[(long long)q * E + e];
        dp[i] += (float)(bal_scale * (double)ce);
      }
      s += p[i] * dp[i];
    }
  }
  s = warp_sum(s);
  const float inv_tau = 1.0f / tau;
#pragma unroll
  for (int i = 0; i < kMaxEPL; ++i) {
    int e = lane + 32 * i;
    const float v = e < E ? p[i] * (dp[i] - s) * inv_tau : 0.f;
    if (e < E) dlogits[(long long)t * E + e] = v;
    if (dL2 && e < Ep) {   // tensor-core operand row [hi | lo | 0] of dlogits (dl_split_kernel's layout)
      const bf16 hi = __float2bfloat16_rn(v);
      dL2[(long long)t * Kp + e] = hi;
      dL2[(long long)t * Kp + Ep + e] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
  }
  if (dL2)
    for (int k = 2 * Ep + lane; k < Kp; k += 32) dL2[(long long)t * Kp + k] = __float2bfloat16_rn(0.f);
}

// The same for E = 16, 32, 64 (E a power of two and Ep == E): lane = four adjacent (token,
// expert) entries of the flat [T, E] arrays (float4 / int4 loads, one 8-byte store of each bf16
// half of dL), E / 4 lanes per token; <p, dp> is a butterfly over the token's E / 4 lanes.  A
// quarter of the threads and memory instructions of the lane-per-expert form (C4: 48 -> 31 us;
// two entries per lane: 38 us).
template <bool PEER = false>
__global__ void __launch_bounds__(256) gate_bwd_quad_kernel(
    const float* __restrict__ dG_row, const int* __restrict__ slot, const float* __restrict__ probs,
    int T_, int E, float tau, float alpha, const int* __restrict__ counts, int count_rows, double bal_scale,
    float* __restrict__ dlogits, bf16* __restrict__ dL2, int Ep, int Kp, int El,
    const __grid_constant__ PeerTable dGp) {
  const int lane = threadIdx.x % 32;
  const long long i0 = 4 * (((long long)blockIdx.x * 8 + threadIdx.x / 32) * 32 + lane);
  const long long t = i0 / E;
  const int e = (int)(i0 % E), G = E / 4;
  const bool ok = t < T_;
  float4 pp = make_float4(0.f, 0.f, 0.f, 0.f);
  int4 rr = make_int4(-1, -1, -1, -1);
  if (ok) {
    pp = *reinterpret_cast<const float4*>(probs + i0);
    rr = *reinterpret_cast<const int4*>(slot + i0);
  }
  const int r4[4] = {rr.x, rr.y, rr.z, rr.w};
  const float p4[4] = {pp.x, pp.y, pp.z, pp.w};
  float dp[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    dp[j] = r4[j] >= 0 ? (PEER ? reinterpret_cast<const float*>(dGp.p[(e + j) / El])[r4[j]] : dG_row[r4[j]]) : 0.f;
  if (alpha > 0.f && ok) {                 // global count of e: the column sum of the count rows
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int cn = 0;
      for (int q = 0; q < count_rows; ++q) cn += counts[(long long)q * E + e + j];
      dp[j] += (float)(bal_scale * (double)cn);
    }
  }
  float sum = (p4[0] * dp[0] + p4[1] * dp[1]) + (p4[2] * dp[2] + p4[3] * dp[3]);
  for (int o = 1; o < G; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (!ok) return;
  const float inv_tau = 1.0f / tau;
  float v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = p4[j] * (dp[j] - sum) * inv_tau;
  *reinterpret_cast<float4*>(dlogits + i0) = make_float4(v[0], v[1], v[2], v[3]);
  if (dL2) {   // tensor-core operand row [hi | lo | 0] of dlogits (dl_split_kernel's layout)
    bf16 h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h[j] = __float2bfloat16_rn(v[j]);
      l[j] = __float2bfloat16_rn(v[j] - __bfloat162float(h[j]));
    }
    bf16* row = dL2 + t * Kp;
    const __nv_bfloat162 h01 = __halves2bfloat162(h[0], h[1]), h23 = __halves2bfloat162(h[2], h[3]);
    const __nv_bfloat162 l01 = __halves2bfloat162(l[0], l[1]), l23 = __halves2bfloat162(l[2], l[3]);
    *reinterpret_cast<uint2*>(row + e) = make_uint2(*reinterpret_cast<const unsigned*>(&h01),
                                                    *reinterpret_cast<const unsigned*>(&h23));
    *reinterpret_cast<uint2*>(row + Ep + e) = make_uint2(*reinterpret_cast<const unsigned*>(&l01),
                                                         *reinterpret_cast<const unsigned*>(&l23));
    for (int k = 2 * Ep + e; k < Kp; k += E) *reinterpret_cast<uint2*>(row + k) = make_uint2(0u, 0u);
  }
}

// out[i] = sum_z part[z][i], fixed order: block = 32 outputs x 8 warps, warp w sums the splits
// z = w, w + 8, ... of its lane's output, the 8 warp sums are added in order w = 0..7
__global__ void __launch_bounds__(256) reduce_splits_kernel(const float* __restrict__ part, int splits, long long n,
                                                           float* __restrict__ out) {
  __shared__ float red[8][32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long i = (long long)blockIdx.x * 32 + lane;
  float acc = 0.f;
  if (i < n)
    for (int z = warp; z < splits; z += 8) acc += part[(long long)z * n + i];
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && i < n) {
    float a = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) a += red[w][lane];
    out[i] = a;
  }
}

// ------------------------------------------------------------------ balance loss
__global__ void colsum_probs_kernel(const float* __restrict__ probs, int T_, int E, float* __restrict__ out) {
  const int e = blockIdx.x;
  __shared__ float red[256];
  float acc = 0.f;
  for (int t = threadIdx.x; t < T_; t += blockDim.x) acc += probs[(long long)t * E + e];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[e] = red[0];
}

__global__ void balance_loss_kernel(const float* __restrict__ colsum, const int* __restrict__ counts, int E,
                                    float alpha, double B, float* __restrict__ loss) {
  if (threadIdx.x != 0) return;
  double acc = 0.0;
  for (int e = 0; e < E; ++e) acc += (double)counts[e] / (B * B) * (double)colsum[e];
  *loss = (float)(alpha * E * acc);
}

}  // namespace

cudaError_t launch_gate(const moe_ctx* c, const void* x, const void* Wg, const float* u, float tau, float thr,
                        int top1, float* probs, int32_t* slot, int32_t* counts, int32_t* near_band,
                        cudaStream_t s) {
  cudaError_t e;
  // the tcgen05 path zeroes counts / near_band in its first kernel (no memset nodes in the step)
  if (c->T > 0 && gate_tc_supported(c)) return gate_tc_forward(c, x, Wg, u, tau, thr, top1, probs, slot, counts, near_band, s);
  if ((e = cudaMemsetAsync(counts, 0, sizeof(int) * c->E, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(near_band, 0, sizeof(int), s)) != cudaSuccess) return e;
  if (c->T == 0) return cudaSuccess;
  if (c->dtype == 1) return launch_gate_typed<bf16>(c, x, Wg, u, tau, thr, top1, probs, slot, counts, near_band, s);
  return launch_gate_typed<float>(c, x, Wg, u, tau, thr, top1, probs, slot, counts, near_band, s);
}

// dx = dlogits W_g^T for the non-tensor-core gate path: fp32 SIMT product into the workspace,
// stored in the activation dtype
__global__ void f32_to_act_kernel(const float* __restrict__ in, long long n, bf16* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

static cudaError_t gate_bwd_impl(const moe_ctx* c, const float* dG_row, const PeerTable* dGp, const int32_t* slot,
                                 const float* probs, const void* x, const void* Wg, float tau, float alpha,
                                 const int32_t* counts, int count_rows, int64_t B_total, float* dWg, float* dlogits,
                                 void* dx, cudaStream_t s) {
  if (c->T == 0) return cudaMemsetAsync(dWg, 0, sizeof(float) * c->d * c->E, s);
  double bal = alpha > 0.f ? (double)alpha * c->E / ((double)B_total * (double)B_total) : 0.0;
  const bool tc = gate_tc_supported(c);
  bf16* dL2 = tc ? reinterpret_cast<bf16*>(gate_dl2_buffer(c)) : nullptr;
  const int Ep = (c->E + 15) / 16 * 16, Kp = (2 * Ep + 63) / 64 * 64;
  PeerTable tab{};
  const bool quad = c->E >= 16 && c->E <= 64 && (c->E & (c->E - 1)) == 0 && Ep == c->E;
  if (quad) {
    // 256 threads = 1024 entries of the flat [T, E] arrays per block
    const unsigned grid = (unsigned)(((long long)c->T * c->E + 1023) / 1024);
    if (dGp) {
      tab = *dGp;
      gate_bwd_quad_kernel<true><<<grid, 256, 0, s>>>(nullptr, slot, probs, c->T, c->E, tau, alpha, counts, count_rows,
                                                      bal, dlogits, dL2, Ep, Kp, c->E_local, tab),
          count_launch();
    } else {
      gate_bwd_quad_kernel<false><<<grid, 256, 0, s>>>(dG_row, slot, probs, c->T, c->E, tau, alpha, counts, count_rows,
                                                       bal, dlogits, dL2, Ep, Kp, c->E_local, tab),
          count_launch();
    }
  } else if (dGp) {
    tab = *dGp;
    gate_bwd_token_kernel<true><<<(c->T + 7) / 8, 256, 0, s>>>(nullptr, slot, probs, c->T, c->E, tau, alpha, counts,
                                                               count_rows, bal, dlogits, dL2, Ep, Kp, c->E_local, tab),
        count_launch();
  } else {
    gate_bwd_token_kernel<false><<<(c->T + 7) / 8, 256, 0, s>>>(dG_row, slot, probs, c->T, c->E, tau, alpha, counts,
                                                                count_rows, bal, dlogits, dL2, Ep, Kp, c->E_local,
                                                                tab),
        count_launch();
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (tc) {
    // the token kernel above just wrote the [hi | lo] bf16 operand rows of dlogits: both
    // tensor-core products of this call use them (nothing is carried to a later call)
    if ((e = gate_tc_dwg(c, x, dlogits, dWg, true, s)) != cudaSuccess) return e;
    return dx ? gate_tc_dx(c, dlogits, Wg, dx, true, s) : cudaSuccess;
  }
  // dWg [d, E] = x^T [d, T] . dlogits [T, E]  (split-K, deterministic reduction)
  SimtGemm g{};
  g.A = x; g.sAm = 1; g.sAk = c->d;
  g.B = dlogits; g.sBk = c->E; g.sBn = 1;
  g.M = c->d; g.N = c->E; g.K = c->T; g.G = 1;
  g.k_split = c->dwg_splits;
  g.sCm = c->E; g.gC = (long long)c->d * c->E;
  g.C = c->dwg_splits > 1 ? (void*)c->part : (void*)dWg;
  if ((e = launch_simt_gemm(g, c->dtype, 0, 0, EPI_F32, s)) != cudaSuccess) return e;
  if (c->dwg_splits > 1) {
    long long n = (long long)c->d * c->E;
    reduce_splits_kernel<<<(unsigned)((n + 31) / 32), 256, 0, s>>>(c->part, c->dwg_splits, n, dWg), count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (!dx) return cudaSuccess;
  // dx [T, d] = dlogits [T, E] . Wg^T  (Wg [d, E] -> B(k=e, n=dd) = Wg[dd*E + e]); fp32 straight
  // into dx for fp32 layers, through the fp32 workspace buffer for bf16 ones
  SimtGemm h{};
  h.A = dlogits; h.sAm = c->E; h.sAk = 1;
  h.B = Wg; h.sBk = 1; h.sBn = c->E;
  h.C = c->dtype == 1 ? (void*)c->dxg : dx; h.sCm = c->d;
  h.M = c->T; h.N = c->d; h.K = c->E; h.G = 1; h.k_split = 1;
  if ((e = launch_simt_gemm(h, 0, c->dtype, 0, EPI_F32, s)) != cudaSuccess) return e;
  if (c->dtype == 1) {
    const long long n = (long long)c->T * c->d;
    const int blocks = (int)((n + 255) / 256 < 8 * c->sm_count ? (n + 255) / 256 : 8 * c->sm_count);
    f32_to_act_kernel<<<blocks, 256, 0, s>>>(c->dxg, n, reinterpret_cast<bf16*>(dx)), count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_gate_bwd(const moe_ctx* c, const float* dG_row, const int32_t* slot, const float* probs,
                            const void* x, const void* Wg, float tau, float alpha, const int32_t* counts,
                            int count_rows, int64_t B_total, float* dWg, float* dlogits, void* dx, cudaStream_t s) {
  return gate_bwd_impl(c, dG_row, nullptr, slot, probs, x, Wg, tau, alpha, counts, count_rows, B_total, dWg, dlogits,
                       dx, s);
}

cudaError_t launch_gate_bwd_peer(const moe_ctx* c, const PeerTable& dGp, const int32_t* slot, const float* probs,
                                 const void* x, const void* Wg, float tau, float alpha, const int32_t* counts,
                                 int count_rows, int64_t B_total, float* dWg, float* dlogits, void* dx,
                                 cudaStream_t s) {
  return gate_bwd_impl(c, nullptr, &dGp, slot, probs, x, Wg, tau, alpha, counts, count_rows, B_total, dWg, dlogits,
                       dx, s);
}

// Steps 2-3 from precomputed fp32 logits, thread per token (kGateBT tokens per block):
// coalesced smem staging of the logits / noise blocks, Gumbel + tau-softmax + decision in one
// thread, coalesced probs / slot writes, per-block expert counts.  Tokens within kRefine of a
// decision boundary are queued for the fp64 gate_token_refine pass (which also counts them).
__global__ void __launch_bounds__(kGateBT) gate_softmax_tpt_kernel(
    const float* __restrict__ logits, const float* __restrict__ u, int T_, int E, float tau, float thr, int top1,
    float* __restrict__ probs, int* __restrict__ slot, int* __restrict__ counts, int* __restrict__ blk_cnt,
    int* __restrict__ near_band, int* __restrict__ flags, int* __restrict__ rq_count, int* __restrict__ rq_list) {
  extern __shared__ float tsm[];
  __shared__ int s_cnt[128];
  __shared__ int s_band;
  __shared__ unsigned s_bits[kGateBT][4];
  const int LP = E + 1;
  float* ls = tsm;                    // [kGateBT][E+1]
  float* us = tsm + kGateBT * LP;     // [kGateBT][E+1]
  const int tid = threadIdx.x;
  const int t0 = blockIdx.x * kGateBT;
  const int ntok = min(kGateBT, T_ - t0);
  for (int i = tid; i < E; i += kGateBT) s_cnt[i] = 0;
  if (tid == 0) s_band = 0;
  for (int i = tid; i < ntok * E; i += kGateBT) {
    ls[(i / E) * LP + (i % E)] = logits[(long long)t0 * E + i];
    us[(i / E) * LP + (i % E)] = u ? u[(long long)t0 * E + i] : 0.5f;
  }
  __syncthreads();
  if (tid < ntok) {
    const int t = t0 + tid;
    float* L = ls + tid * LP;
    const float* uu = us + tid * LP;
    float mx = -INFINITY;
    bool bad = false;
    for (int e = 0; e < E; ++e) {
      const float Lv = L[e];
      if (!isfinite(Lv)) bad = true;
      const float zeta = u ? -logf(-logf(uu[e])) : 0.f;
      const float z = (Lv + zeta) / tau;
      L[e] = z;
      mx = fmaxf(mx, z);
    }
    if (bad && atomicOr(&flags[0], kFlagNonFinite) == 0) flags[1] = t;
    float sum = 0.f;
    for (int e = 0; e < E; ++e) {
      const float ex = expf(L[e] - mx);
      L[e] = ex;
      sum += ex;
    }
    const float inv = 1.0f / sum;
    bool any_pass = false, near = false;
    float best = -1.f, second = -1.f;
    int am = 0;
    for (int e = 0; e < E; ++e) {
      const float pe = L[e] * inv;
      L[e] = pe;
      if (pe > thr) any_pass = true;
      if (fabsf(pe - thr) < kRefine) near = true;
      if (pe > best) { second = best; best = pe; am = e; }
      else if (pe > second) second = pe;
    }
    const bool argmax_decided = top1 || !any_pass;
    if (top1) near = false;
    if (argmax_decided && best - second < kRefine) near = true;
    unsigned b0 = 0u, b1 = 0u, b2 = 0u, b3 = 0u;
    if (near) {
      rq_list[atomicAdd(rq_count, 1)] = t;      // decided (and counted) by gate_refine_kernel
    } else {
      bool in_band = false;
      for (int e = 0; e < E; ++e) {
        const bool sel = argmax_decided ? (e == am) : (L[e] > thr);
        if (sel) {
          const unsigned bit = 1u << (e & 31);
          if (e < 32) b0 |= bit; else if (e < 64) b1 |= bit; else if (e < 96) b2 |= bit; else b3 |= bit;
          atomicAdd(&s_cnt[e], 1);
        }
        if (!argmax_decided && fabsf(L[e] - thr) < kBand) in_band = true;
      }
      if (argmax_decided) in_band = (best - second) < kBand;
      if (in_band) atomicAdd(&s_band, 1);
    }
    s_bits[tid][0] = b0; s_bits[tid][1] = b1; s_bits[tid][2] = b2; s_bits[tid][3] = b3;
  }
  __syncthreads();
  for (int i = tid; i < ntok * E; i += kGateBT) {
    const int r = i / E, e = i % E;
    probs[(long long)t0 * E + i] = ls[r * LP + e];
    slot[(long long)t0 * E + i] = ((s_bits[r][e >> 5] >> (e & 31)) & 1u) ? 0 : -1;
  }
  for (int e = tid; e < E; e += kGateBT) {
    const int c = s_cnt[e];
    blk_cnt[(long long)e * gridDim.x + blockIdx.x] = c;
    if (c) atomicAdd(&counts[e], c);
  }
  if (tid == 0 && s_band) atomicAdd(near_band, s_band);
}

cudaError_t launch_gate_softmax_tpt(const moe_ctx* c, const float* logits, const float* u, float tau, float thr,
                                    int top1, float* probs, int32_t* slot, int32_t* counts, int32_t* near_band,
                                    cudaStream_t s) {
  const size_t smem = sizeof(float) * 2 * kGateBT * (c->E + 1);
  cudaError_t e = cudaFuncSetAttribute(gate_softmax_tpt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  gate_softmax_tpt_kernel<<<c->nblk, kGateBT, smem, s>>>(logits, u, c->T, c->E, tau, thr, top1, probs, slot, counts,
                                                         c->blk_cnt, near_band, c->flags, c->rq, c->rq + 1),
      count_launch();
  return cudaGetLastError();
}

cudaError_t launch_reduce_splits(const float* part, int splits, long long n, float* out, cudaStream_t s) {
  reduce_splits_kernel<<<(unsigned)((n + 31) / 32), 256, 0, s>>>(part, splits, n, out), count_launch();
  return cudaGetLastError();
}

cudaError_t launch_balance_loss(const moe_ctx* c, const float* probs, const int32_t* counts, float alpha,
                                int64_t B_total, float* loss, cudaStream_t s) {
  colsum_probs_kernel<<<c->E, 256, 0, s>>>(probs, c->T, c->E, c->colsum), count_launch();
  balance_loss_kernel<<<1, 32, 0, s>>>(c->colsum, counts, c->E, alpha, (double)B_total, loss), count_launch();
  return cudaGetLastError();
}

}  // namespace moe
