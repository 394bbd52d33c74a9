// gemm_simt.cu -- CUDA-core (FFMA) grouped GEMM with fp32 accumulation.
//
// Used for the fp32 configuration (C1), where tf32 tensor cores would miss the
// 1e-4 tolerance (SURVEY §2.3 note), and for the small gate contractions until their
// tensor-core versions land.  64x64 output tile, BK = 16, 256 threads, 4x4 per thread.
#include "common.cuh"
#include "internal.h"

namespace moe {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename TX> __device__ __forceinline__ float ldf(const TX* p, long long i) { return to_f32(p[i]); }

template <typename TA, typename TB, typename TO, int EPI>
__global__ void __launch_bounds__(256) simt_gemm_kernel(SimtGemm g) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int n0 = blockIdx.x * BN;
  long long m0 = (long long)blockIdx.y * BM;
  int grp = 0;
  long long k_begin = 0, k_end = g.K;
  long long m_end = g.M;
  if (g.m_off) {
    const long long R = g.m_off[g.G];
    if (m0 >= R) return;
    // tile lies inside one 128-aligned segment: find it
    int lo = 0, hi = g.G - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (g.m_off[mid] <= m0) lo = mid; else hi = mid - 1;
    }
    grp = lo;
    m_end = g.m_off[grp + 1];
  } else if (g.k_off) {
    grp = blockIdx.z;
    k_begin = g.k_off[grp];
    k_end = g.k_off[grp + 1];
  } else if (g.k_split > 1) {
    long long chunk = ((g.K + g.k_split - 1) / g.k_split + BK - 1) / BK * BK;
    k_begin = (long long)blockIdx.z * chunk;
    k_end = min((long long)g.K, k_begin + chunk);
    grp = blockIdx.z;
  }
  const TA* A = reinterpret_cast<const TA*>(g.A);
  const TB* B = reinterpret_cast<const TB*>(g.B) + (long long)grp * g.gB;
  const bool a_mcontig = (g.sAm == 1);
  const bool b_ncontig = (g.sBn == 1);

  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (long long k0 = k_begin; k0 < k_end; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int idx = tid + i * 256;
      int r, kk;
      if (a_mcontig) { r = idx % BM; kk = idx / BM; } else { r = idx / BK; kk = idx % BK; }
      long long m = m0 + r, k = k0 + kk;
      As[kk][r] = (m < m_end && k < k_end) ? ldf(A, m * g.sAm + k * g.sAk) : 0.f;
      int c, kb;
      if (b_ncontig) { c = idx % BN; kb = idx / BN; } else { c = idx / BK; kb = idx % BK; }
      long long n = n0 + c, k2 = k0 + kb;
      Bs[kb][c] = (n < g.N && k2 < k_end) ? ldf(B, k2 * g.sBk + n * g.sBn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  long long cbase = 0;
  if (g.k_off || (!g.m_off && g.k_split > 1)) cbase = (long long)grp * g.gC;
  const TO* bias = reinterpret_cast<const TO*>(g.bias);
  if (bias) bias += (long long)grp * g.gBias;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    long long m = m0 + ty * 4 + i;
    if (m >= m_end) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      long long ci = cbase + m * g.sCm + n;
      float v = acc[i][j];
      if (EPI == EPI_F32) {
        reinterpret_cast<float*>(g.C)[ci] = v;
      } else if (EPI == EPI_T) {
        reinterpret_cast<TO*>(g.C)[ci] = from_f32<TO>(v);
      } else if (EPI == EPI_BIAS_T) {
        reinterpret_cast<TO*>(g.C)[ci] = from_f32<TO>(v + to_f32(bias[n]));
      } else if (EPI == EPI_BIAS_GELU) {
        // pre-activation a in fp32; store gp = GELU'(a) (for the backward) and h = GELU(a)
        const float a = v + to_f32(bias[n]);
        if (g.C) reinterpret_cast<TO*>(g.C)[ci] = from_f32<TO>(gelu_prime_f(a));
        reinterpret_cast<TO*>(g.C2)[ci] = from_f32<TO>(gelu_f(a));
      } else if (EPI == EPI_GELU_BWD) {
        const float gp = to_f32(reinterpret_cast<const TO*>(g.aux)[ci]);   // saved GELU'(a)
        reinterpret_cast<TO*>(g.C)[ci] = from_f32<TO>(v * gp);
      }
    }
  }
}

template <typename TA, typename TB, typename TO>
cudaError_t launch_typed(const SimtGemm& g, int epi, cudaStream_t s) {
  dim3 grid((g.N + BN - 1) / BN, 1, 1);
  if (g.m_off) {
    grid.y = (unsigned)g.m_tiles;
  } else {
    grid.y = (g.M + BM - 1) / BM;
    if (g.k_off) grid.z = g.G;
    else if (g.k_split > 1) grid.z = g.k_split;
  }
  if (grid.y == 0 || grid.x == 0) return cudaSuccess;
  switch (epi) {
    case EPI_F32: simt_gemm_kernel<TA, TB, TO, EPI_F32><<<grid, 256, 0, s>>>(g), count_launch(); break;
    case EPI_T: simt_gemm_kernel<TA, TB, TO, EPI_T><<<grid, 256, 0, s>>>(g), count_launch(); break;
    case EPI_BIAS_T: simt_gemm_kernel<TA, TB, TO, EPI_BIAS_T><<<grid, 256, 0, s>>>(g), count_launch(); break;
    case EPI_BIAS_GELU: simt_gemm_kernel<TA, TB, TO, EPI_BIAS_GELU><<<grid, 256, 0, s>>>(g), count_launch(); break;
    case EPI_GELU_BWD: simt_gemm_kernel<TA, TB, TO, EPI_GELU_BWD><<<grid, 256, 0, s>>>(g), count_launch(); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Per-group column sums (bias gradients), deterministic two-phase reduction.
// Phase 1: block (column block of 256, split s, group g); lane = 8 columns (16-byte loads),
// warp w sums rows r0 + w, r0 + w + 8, ... of its split; warps combined in fixed order.
template <typename TI>
__global__ void __launch_bounds__(256) colsum_part_kernel(const TI* __restrict__ X, int N, const int* __restrict__ m_off,
                                                         int S, int shift, float* __restrict__ part) {
  constexpr int V = Vec16<TI>::N;                 // elements per 16-byte vector
  constexpr int COLS = 32 * V;                     // columns per block
  __shared__ float red[8][COLS];
  const int g = blockIdx.z, s = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n0 = blockIdx.x * COLS + lane * V;
  const int off0 = m_off[g] >> shift, len = (m_off[g + 1] >> shift) - off0;   // rows of X = m_off >> shift
  const int per = (len + S - 1) / S;
  const int r0 = off0 + s * per, r1 = min(off0 + len, r0 + per);
  float acc[V];
#pragma unroll
  for (int k = 0; k < V; ++k) acc[k] = 0.f;
  if (n0 < N) {
    // rows r, r + 8, r + 16, r + 24 in flight together (a split is often only a few rows per
    // warp: the ragged tail is predicated, not a serial loop); rows are added in ascending order
    for (int r = r0 + warp; r < r1; r += 32) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        q[u] = r + 8 * u < r1 ? ld_nc_v4(X + (long long)(r + 8 * u) * N + n0) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float f[V];
        unpack16(q[u], f, TI());
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] += f[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < V; ++k) red[warp][lane * V + k] = acc[k];
  __syncthreads();
  for (int c = threadIdx.x; c < COLS; c += 256) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][c];
    const int n = blockIdx.x * COLS + c;
    if (n < N) part[((long long)g * S + s) * N + n] = t;
  }
}

// out[g][n] = sum_s part[g][s][n] (few splits): thread per column, splits in order
__global__ void colsum_final_seq_kernel(const float* __restrict__ part, int N, int S, float* __restrict__ out) {
  const int g = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float t = 0.f;
  for (int s = 0; s < S; ++s) t += part[((long long)g * S + s) * N + n];
  out[(long long)g * N + n] = t;
}

// out[g][n] = sum_s part[g][s][n] (many splits): block = 32 columns x 8 warps; warp w sums the splits
// s = w, w + 8, ... (ascending) of its lane's column, then the 8 warp sums are added in
// order w = 0..7 (fixed order, deterministic; 8 loads in flight per column instead of S).
__global__ void __launch_bounds__(256) colsum_final_kernel(const float* __restrict__ part, int N, int S,
                                                          float* __restrict__ out) {
  __shared__ float red[8][32];
  const int g = blockIdx.y, warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n = blockIdx.x * 32 + lane;
  float t = 0.f;
  if (n < N)
    for (int sp = warp; sp < S; sp += 8) t += part[((long long)g * S + sp) * N + n];
  red[warp][lane] = t;
  __syncthreads();
  if (warp == 0 && n < N) {
    float a = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) a += red[w][lane];
    out[(long long)g * N + n] = a;
  }
}

}  // namespace

// the second phase of the column sums: warp-split over the partials when there are many
static void launch_final(const float* part, int N, int S, int G, float* out, cudaStream_t s) {
  if (S >= 16)
    colsum_final_kernel<<<dim3((N + 31) / 32, G), 256, 0, s>>>(part, N, S, out), count_launch();
  else
    colsum_final_seq_kernel<<<dim3((N + 255) / 256, G), 256, 0, s>>>(part, N, S, out), count_launch();
}

cudaError_t launch_simt_gemm(const SimtGemm& g, int ta, int tb, int tout, int epi, cudaStream_t s) {
  if (ta == 0 && tb == 0) return launch_typed<float, float, float>(g, epi, s);
  if (ta == 1 && tb == 1) {
    if (tout == 1) return launch_typed<bf16, bf16, bf16>(g, epi, s);
    return launch_typed<bf16, bf16, float>(g, EPI_F32, s);
  }
  if (ta == 1 && tb == 0) return launch_typed<bf16, float, float>(g, EPI_F32, s);
  return launch_typed<float, bf16, float>(g, EPI_F32, s);
}

// db1[g][n] = sum over the 32-row blocks of group g of part[rb][n]: the same two-phase fixed-order
// reduction as the column sums, over the [R/32][N] fp32 partial rows (m_off >> 5).
cudaError_t launch_db1_reduce(const float* part, int N, const int* m_off, int G, float* out, float* part2,
                              long long R_cap, cudaStream_t s) {
  if (G == 0 || N == 0) return cudaSuccess;
  // splits per expert: ~32 partial rows (of 32 token rows each) per split, at most kColsumSplits
  long long per = R_cap / 32 / G;
  int S = (int)((per + 31) / 32);
  S = S < 1 ? 1 : (S > kColsumSplits ? kColsumSplits : S);
  colsum_part_kernel<float><<<dim3((N + 127) / 128, S, G), 256, 0, s>>>(part, N, m_off, S, 5, part2), count_launch();
  launch_final(part2, N, S, G, out, s);
  return cudaGetLastError();
}

cudaError_t launch_colsum_grouped(const void* X, int tin, int N, const int* m_off, int G, float* out,
                                  float* part, cudaStream_t s) {
  if (G == 0 || N == 0) return cudaSuccess;
  const int S = kColsumSplits;
  const int cols = tin == 0 ? 128 : 256;
  dim3 g1((N + cols - 1) / cols, S, G);
  if (tin == 0)
    colsum_part_kernel<float><<<g1, 256, 0, s>>>(reinterpret_cast<const float*>(X), N, m_off, S, 0, part), count_launch();
  else
    colsum_part_kernel<bf16><<<g1, 256, 0, s>>>(reinterpret_cast<const bf16*>(X), N, m_off, S, 0, part), count_launch();
  launch_final(part, N, S, G, out, s);
  return cudaGetLastError();
}

cudaError_t launch_colsum_final(const float* part, int N, int S, int G, float* out, cudaStream_t s) {
  if (G == 0 || N == 0) return cudaSuccess;
  launch_final(part, N, S, G, out, s);
  return cudaGetLastError();
}

}  // namespace moe
