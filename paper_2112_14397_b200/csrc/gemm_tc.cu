// gemm_tc.cu -- persistent, warp-specialised tcgen05 grouped GEMM for the expert FFN
// (step 5 and B5).  bf16 operands staged by TMA (128-byte swizzle) into a 4-stage
// shared-memory ring, tcgen05.mma (M=128, N=256, K=16) accumulating in TMEM (two
// 256-column accumulators so the epilogue of tile i overlaps the mainloop of tile i+1),
// tcgen05.ld epilogue with the fused bias / GELU / GELU' / fp32-store variants.
//
// Roles (192 threads):  warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
//                       warps 2..5 = epilogue (thread = accumulator row).
// Scheduling: static round-robin over tiles; every role walks the same tile sequence.
//   ROWS mode  (ragged M): tiles = (offsets[G]/128) x ceil(N/256); group found from the
//              device offsets[] (segments are 128-row aligned, so a tile never straddles).
//   KGRP mode  (ragged K, weight gradients): tiles = G x ceil(M/128) x ceil(N/256);
//              K range of group g = [offsets[g], offsets[g+1]); empty groups store zeros.
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"

namespace moe {

namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;          // 16 KB
constexpr int B_BYTES = BN * BK * 2;          // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;                // 2 accumulators x 256 fp32 columns
constexpr int NUM_THREADS = 192;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers, offsets*/;
constexpr int MAX_G = 128;

enum TcEpi { TEPI_BIAS_GELU = 0, TEPI_BIAS = 1, TEPI_GELU_BWD = 2, TEPI_STORE = 3, TEPI_F32 = 4 };

struct TcParams {
  int kgrp;               // 0 = ragged M (ROWS), 1 = ragged K (KGRP)
  int G;
  const int* offsets;     // [G+1]
  int M, N, K;            // ROWS: N, K used; KGRP: M, N used
  int m_tiles_cap;        // ROWS: R_cap / 128
  int b_group_rows;       // ROWS: B tensor-map row offset of group g = g * b_group_rows
  void* out;              // row-major, pitch ldo elements
  long long ldo;
  long long out_g;        // KGRP: out + g * out_g
  void* out2;             // TEPI_BIAS_GELU: h
  const void* bias;       // + g * bias_g
  long long bias_g;
  const void* aux;        // TEPI_GELU_BWD: a (pitch ldo)
};

struct Tile {
  int g, m0, n0, kb0, nkb;
};

template <bool KGRP>
__device__ __forceinline__ bool decode_tile(const TcParams& p, const int* s_off, int t, int n_tiles, Tile& tl) {
  if (!KGRP) {
    const int mt = t / n_tiles, nt = t - mt * n_tiles;
    tl.m0 = mt * BM;
    tl.n0 = nt * BN;
    int lo = 0, hi = p.G - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= tl.m0) lo = mid; else hi = mid - 1;
    }
    tl.g = lo;
    tl.kb0 = 0;
    tl.nkb = (p.K + BK - 1) / BK;
  } else {
    const int m_tiles = (p.M + BM - 1) / BM;
    const int per_g = m_tiles * n_tiles;
    tl.g = t / per_g;
    const int r = t - tl.g * per_g;
    const int mt = r / n_tiles, nt = r - mt * n_tiles;
    tl.m0 = mt * BM;
    tl.n0 = nt * BN;
    tl.kb0 = s_off[tl.g] / BK;
    tl.nkb = (s_off[tl.g + 1] - s_off[tl.g]) / BK;
  }
  return tl.nkb > 0;
}

template <int EPI, bool A_MN, bool B_MN, bool KGRP>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned ring (SWIZZLE_128B atoms)
  const uint32_t raw_u32 = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_u32 & 1023)) & 1023);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* s_off = reinterpret_cast<int*>(s_tmem + 4);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i <= p.G && i <= MAX_G; i += NUM_THREADS) s_off[i] = p.offsets[i];
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull_bar[a], 1);
      tc::mbar_init(&tempty_bar[a], 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) {
    tc::tmem_alloc(s_tmem, TMEM_COLS);
    tc::tmem_relinquish();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  const int n_tiles = (p.N + BN - 1) / BN;
  int total;
  if (!KGRP) {
    int R = s_off[p.G];
    const int cap = p.m_tiles_cap * BM;
    if (R > cap) R = cap;
    total = (R / BM) * n_tiles;
  } else {
    total = p.G * ((p.M + BM - 1) / BM) * n_tiles;
  }

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        Tile tl;
        if (!decode_tile<KGRP>(p, s_off, t, n_tiles, tl)) continue;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          tc::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          tc::mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          const int k = (tl.kb0 + kb) * BK;
          if (!A_MN) {
            tc::tma_load_2d(sa, &tmA, &full_bar[stage], k, tl.m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c) tc::tma_load_2d(sa + c * 8192, &tmA, &full_bar[stage], tl.m0 + c * 64, k);
          }
          const int brow = KGRP ? 0 : tl.g * p.b_group_rows;
          if (!B_MN) {
            tc::tma_load_2d(sb, &tmB, &full_bar[stage], k, brow + tl.n0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tc::tma_load_2d(sb + c * 8192, &tmB, &full_bar[stage], tl.n0 + c * 64, brow + k);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t smem_base = tc::smem_u32(smem);
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        Tile tl;
        if (!decode_tile<KGRP>(p, s_off, t, n_tiles, tl)) continue;
        tc::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          tc::mbar_wait(&full_bar[stage], phase);
          tc::tc_fence_after();
          const uint32_t sa = smem_base + stage * STAGE_BYTES;
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major SW128: +32 B per K=16 step, SBO = 1024 (8 rows x 128 B)
            // MN-major SW128: +2048 B per K=16 step (16 rows x 128 B), LBO = 8 KB (64-wide MN chunk), SBO = 1024
            const uint64_t ad = A_MN ? tc::smem_desc_sw128(sa + k * 2048, 8192, 1024)
                                     : tc::smem_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? tc::smem_desc_sw128(sb + k * 2048, 8192, 1024)
                                     : tc::smem_desc_sw128(sb + k * 32, 16, 1024);
            tc::mma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          tc::mma_commit(&empty_bar[stage]);           // frees the smem slot when these MMAs finish
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit(&tfull_bar[acc]);                // accumulator ready for the epilogue
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int sub = warp & 3;                          // TMEM lane quarter this warp may access
    const int row_in_tile = sub * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      Tile tl;
      const bool nonempty = decode_tile<KGRP>(p, s_off, t, n_tiles, tl);
      const long long row = (long long)tl.m0 + row_in_tile;
      const bool row_ok = KGRP ? (row < p.M) : true;
      if (!nonempty) {
        // KGRP only: empty expert -> zero gradient tile
        if (row_ok) {
          float* o = reinterpret_cast<float*>(p.out) + (long long)tl.g * p.out_g + row * p.ldo;
          for (int c = 0; c < BN; c += 4)
            if (tl.n0 + c < p.N) *reinterpret_cast<float4*>(o + tl.n0 + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        continue;
      }
      tc::mbar_wait(&tfull_bar[acc], acc_phase);
      tc::tc_fence_after();
      const uint32_t t_row = tmem_base + acc * BN + ((uint32_t)(sub * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tc::tmem_ld32(t_row + c, r);
        tc::tmem_ld_wait();
        const int n = tl.n0 + c;
        if (n >= p.N || !row_ok) continue;
        if (EPI == TEPI_F32) {
          float* o = reinterpret_cast<float*>(p.out) + (long long)tl.g * p.out_g + row * p.ldo + n;
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(o + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                            __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        } else {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          bf16* o = reinterpret_cast<bf16*>(p.out) + row * p.ldo + n;
          if (EPI == TEPI_BIAS_GELU || EPI == TEPI_BIAS) {
            const bf16* bp = reinterpret_cast<const bf16*>(p.bias) + (long long)tl.g * p.bias_g + n;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float b[8];
              unpack16(ld_v4(bp + q * 8), b, bf16());
#pragma unroll
              for (int j = 0; j < 8; ++j) v[q * 8 + j] += b[j];
            }
          }
          if (EPI == TEPI_BIAS_GELU) {
            bf16* o2 = reinterpret_cast<bf16*>(p.out2) + row * p.ldo + n;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              st_v4(o + q * 8, pack16(v + q * 8, bf16()));
              float hq[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) hq[j] = gelu_f(v[q * 8 + j]);
              st_v4(o2 + q * 8, pack16(hq, bf16()));
            }
          } else if (EPI == TEPI_GELU_BWD) {
            const bf16* ap = reinterpret_cast<const bf16*>(p.aux) + row * p.ldo + n;
            uint4 araw[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) araw[q] = ld_v4(ap + q * 8);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float a[8];
              unpack16(araw[q], a, bf16());
#pragma unroll
              for (int j = 0; j < 8; ++j) v[q * 8 + j] *= gelu_prime_f(a[j]);
              st_v4(o + q * 8, pack16(v + q * 8, bf16()));
            }
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) st_v4(o + q * 8, pack16(v + q * 8, bf16()));
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D bf16 tensor map over a row-major [rows, cols] matrix with row pitch `pitch` elements;
// box = {box_cols (inner), box_rows}, 128-byte swizzle (box_cols * 2 must be 128).
bool make_map(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long pitch, int box_cols,
              int box_rows) {
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int EPI, bool A_MN, bool B_MN, bool KGRP>
cudaError_t launch_tc(const CUtensorMap& a, const CUtensorMap& b, const TcParams& p, int tiles_upper, int sms,
                      cudaStream_t s) {
  auto k = tc_gemm_kernel<EPI, A_MN, B_MN, KGRP>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int grid = tiles_upper < sms ? tiles_upper : sms;
  if (grid <= 0) return cudaSuccess;
  k<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(a, b, p), count_launch();
  return cudaGetLastError();
}

}  // namespace

bool tc_available() { return encode_fn() != nullptr; }

// ---------------------------------------------------------------- step 5 / B5 on tensor cores
cudaError_t tc_expert_ffn(const moe_ctx* c, const void* x_perm, const int32_t* offsets, int64_t R_cap,
                          const void* W1, const void* b1, const void* W2, const void* b2, void* a, void* h,
                          void* e_out, cudaStream_t s) {
  const int d = c->d, f = c->f, El = c->E_local;
  if (R_cap == 0) return cudaSuccess;
  CUtensorMap mA, mB;
  TcParams p{};
  p.kgrp = 0; p.G = El; p.offsets = offsets; p.m_tiles_cap = (int)(R_cap / BM);
  // GEMM1: a = x_perm W1^T + b1, h = GELU(a)      A [R, d] K-major, B = W1 [El*f, d] K-major
  if (!make_map(&mA, x_perm, R_cap, d, d, 64, BM) || !make_map(&mB, W1, (long long)El * f, d, d, 64, BN))
    return cudaErrorInvalidValue;
  p.N = f; p.K = d; p.b_group_rows = f;
  p.out = a; p.out2 = h; p.ldo = f; p.bias = b1; p.bias_g = f;
  cudaError_t e = launch_tc<TEPI_BIAS_GELU, false, false, false>(mA, mB, p, p.m_tiles_cap * ((f + BN - 1) / BN),
                                                                  c->sm_count, s);
  if (e != cudaSuccess) return e;
  // GEMM2: e_out = h W2^T + b2                     A [R, f] K-major, B = W2 [El*d, f] K-major
  if (!make_map(&mA, h, R_cap, f, f, 64, BM) || !make_map(&mB, W2, (long long)El * d, f, f, 64, BN))
    return cudaErrorInvalidValue;
  p.N = d; p.K = f; p.b_group_rows = d;
  p.out = e_out; p.out2 = nullptr; p.ldo = d; p.bias = b2; p.bias_g = d;
  return launch_tc<TEPI_BIAS, false, false, false>(mA, mB, p, p.m_tiles_cap * ((d + BN - 1) / BN), c->sm_count, s);
}

cudaError_t tc_expert_ffn_bwd(const moe_ctx* c, const void* d_eout, const void* x_perm, const void* a,
                              const void* h, const int32_t* offsets, int64_t R_cap, const void* W1,
                              const void* W2, void* da, void* dx_perm, float* dW1, float* dW2, cudaStream_t s) {
  const int d = c->d, f = c->f, El = c->E_local;
  CUtensorMap mA, mB;
  cudaError_t e;
  if (R_cap == 0) {   // no rows at all: every expert gradient is zero
    if ((e = cudaMemsetAsync(dW1, 0, sizeof(float) * El * f * d, s)) != cudaSuccess) return e;
    return cudaMemsetAsync(dW2, 0, sizeof(float) * El * d * f, s);
  }
  {
    TcParams p{};
    p.kgrp = 0; p.G = El; p.offsets = offsets; p.m_tiles_cap = (int)(R_cap / BM);
    // dgrad2: da = (d_eout W2_e) (.) GELU'(a)   A = d_eout [R, d] K-major; B(k=d, n=f) = W2 [El*d, f] MN-major
    if (!make_map(&mA, d_eout, R_cap, d, d, 64, BM) || !make_map(&mB, W2, (long long)El * d, f, f, 64, 64))
      return cudaErrorInvalidValue;
    p.N = f; p.K = d; p.b_group_rows = d;
    p.out = da; p.ldo = f; p.aux = a;
    e = launch_tc<TEPI_GELU_BWD, false, true, false>(mA, mB, p, p.m_tiles_cap * ((f + BN - 1) / BN), c->sm_count, s);
    if (e != cudaSuccess) return e;
    // dgrad1: dx_perm = da W1_e                 A = da [R, f] K-major; B(k=f, n=d) = W1 [El*f, d] MN-major
    if (!make_map(&mA, da, R_cap, f, f, 64, BM) || !make_map(&mB, W1, (long long)El * f, d, d, 64, 64))
      return cudaErrorInvalidValue;
    p.N = d; p.K = f; p.b_group_rows = f;
    p.out = dx_perm; p.ldo = d; p.aux = nullptr;
    e = launch_tc<TEPI_STORE, false, true, false>(mA, mB, p, p.m_tiles_cap * ((d + BN - 1) / BN), c->sm_count, s);
    if (e != cudaSuccess) return e;
  }
  // wgrad2: dW2_e [d, f] = d_eout_e^T h_e       A(m=d, k=row) = d_eout MN-major; B(k=row, n=f) = h MN-major
  const long long rows = R_cap;
  TcParams q{};
  q.kgrp = 1; q.G = El; q.offsets = offsets;
  if (!make_map(&mA, d_eout, rows, d, d, 64, 64) || !make_map(&mB, h, rows, f, f, 64, 64))
    return cudaErrorInvalidValue;
  q.M = d; q.N = f; q.out = dW2; q.ldo = f; q.out_g = (long long)d * f;
  e = launch_tc<TEPI_F32, true, true, true>(mA, mB, q, El * ((d + BM - 1) / BM) * ((f + BN - 1) / BN), c->sm_count, s);
  if (e != cudaSuccess) return e;
  // wgrad1: dW1_e [f, d] = da_e^T x_perm_e      A(m=f, k=row) = da MN-major; B(k=row, n=d) = x_perm MN-major
  if (!make_map(&mA, da, rows, f, f, 64, 64) || !make_map(&mB, x_perm, rows, d, d, 64, 64))
    return cudaErrorInvalidValue;
  q.M = f; q.N = d; q.out = dW1; q.ldo = d; q.out_g = (long long)f * d;
  return launch_tc<TEPI_F32, true, true, true>(mA, mB, q, El * ((f + BM - 1) / BM) * ((d + BN - 1) / BN), c->sm_count, s);
}

}  // namespace moe
