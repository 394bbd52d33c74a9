// gemm_gate_tc.cu -- tcgen05 kernels for the skinny gate contractions (bf16 path):
//
//   GATE  L = x W_g                [T, E]   M = 128 tokens / CTA, N = Ep (E padded to 16), K = d
//         (E % 16 != 0: logits to HBM, steps 2-3 in gate_softmax_tpt_kernel + gate_refine_kernel;
//          E % 16 == 0 uses the persistent fused kernel below, steps 1-3 in one launch)
//   DWG   dW_g = x^T dL                [d, E]   M = 128 of d, N = Kp, K = T split over CTAs
//   (the third, dL W_g^T [T, d], runs on the expert GEMM's dense STORE path: gate_tc_dx)
//
// One tile per CTA (no persistence), cta_group::1 tcgen05.mma (M = 128), TMA-fed 4-stage
// ring, single elected MMA thread, 4 epilogue warps reading TMEM with tcgen05.ld.
//
// Precision.  x and W_g products are exact in fp32; the logits must carry ~1 ulp of error
// (1e-5 probs at tau = 0.05-0.1), so GATE accumulates NG contiguous K ranges into NG separate
// TMEM column blocks and the epilogue adds them with TwoSum.  dL (fp32) enters the tensor
// core as a hi + lo pair of bf16 values (dL2 = [hi | lo], K or N doubled), which keeps the
// products near fp32 accuracy.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include "common.cuh"
#include "gate_token.cuh"
#include "internal.h"
#include "tc_ptx.cuh"

namespace moe {

namespace tcgate {

constexpr int BM = 128, BK = 64;
// GATE: 2 stages (2 CTAs / SM; the idle ring then holds the noise block)
template <int MODE> struct Stages { static constexpr int N = MODE == 2 ? 4 : 2; };
template <int MODE> struct Threads { static constexpr int N = 64 + 128; };
// warp 0 TMA, warp 1 MMA + TMEM alloc, then 4 epilogue warps
enum Mode { GATE = 0, DWG = 2 };

struct Params {
  int mode;
  int T, d, E, Ep, Kp;
  int ng;              // GATE: number of K groups (TMEM column blocks of Ep)
  int kb_per_group;    // GATE
  int tmem_cols;
  int split_rows;      // DWG: K rows per split (multiple of BK)
  // GATE
  const bf16* x;
  const bf16* Wg;      // [d, E] (fp64 refine)
  const float* u;
  float tau, thr;
  int top1;
  float* probs;
  int* slot;
  int* counts;
  int* blk_cnt;        // [E][nblk]
  int* near_band;
  int* flags;
  int* rq_count;       // deferred (near-boundary) tokens -> gate_refine_kernel
  int* rq_list;
  float* logits;       // GATE output [T, E] fp32
  // DWG
  float* part;         // [splits, d, E]
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(Threads<MODE>::N) gate_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                                                             const __grid_constant__ CUtensorMap tmB, Params p) {
  constexpr int STAGES = Stages<MODE>::N;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_u32 & 1023)) & 1023);
  // operand bytes per stage
  const int a_bytes = BM * BK * 2;
  const int bn = MODE == GATE ? p.Ep : p.Kp;
  const int b_bytes = bn * BK * 2;
  const int stage_bytes = a_bytes + ((b_bytes + 1023) & ~1023);
  uint8_t* tail = smem + STAGES * stage_bytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(tail);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* done_bar = empty_bar + STAGES;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(done_bar + 1);
  int* s_cnt = reinterpret_cast<int*>(s_tmem + 4);    // [128] expert counts (GATE)
  int* s_band = s_cnt + 128;
  float* s_misc = reinterpret_cast<float*>(s_band + 4);   // GATE logits [128][E+1]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // tile coordinates
  int m0 = 0, n0 = 0, kb0 = 0, nkb = 0;
  if (MODE == GATE) {
    m0 = blockIdx.x * BM; nkb = (p.d + BK - 1) / BK;
  } else {
    m0 = blockIdx.x * BM;                     // rows of dW_g (d index)
    kb0 = blockIdx.y * (p.split_rows / BK);
    const int kb_end = min((p.T + BK - 1) / BK, kb0 + p.split_rows / BK);
    nkb = max(0, kb_end - kb0);
  }

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    tc::mbar_init(done_bar, 1);
    tc::fence_mbar_init();
  }
  if (MODE == GATE) {
    for (int i = threadIdx.x; i < 128; i += Threads<MODE>::N) s_cnt[i] = 0;
    if (threadIdx.x == 0) s_band[0] = 0;
  }
  if (warp == 1) tc::tmem_alloc(s_tmem, p.tmem_cols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * stage_bytes;
        uint8_t* sb = sa + a_bytes;
        const int k = (kb0 + kb) * BK;
        tc::mbar_arrive_expect_tx(&full_bar[stage], a_bytes + b_bytes);
        if (MODE != DWG) {
          tc::tma_load_2d(sa, &tmA, &full_bar[stage], k, m0);              // A K-major [rows, K]
          tc::tma_load_2d(sb, &tmB, &full_bar[stage], k, n0);              // B K-major [N rows, K]
        } else {
          tc::tma_load_2d(sa, &tmA, &full_bar[stage], m0, k);              // A = x MN-major, 2 x 64 chunks
          tc::tma_load_2d(sa + 8192, &tmA, &full_bar[stage], m0 + 64, k);
          for (int c = 0; c < bn / 64; ++c)                                 // B = dL2 MN-major
            tc::tma_load_2d(sb + c * 8192, &tmB, &full_bar[stage], c * 64, k);
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(BM, bn, MODE == DWG ? 1 : 0, MODE == DWG ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t smem_base = tc::smem_u32(smem);
      for (int kb = 0; kb < nkb; ++kb) {
        tc::mbar_wait(&full_bar[stage], phase);
        tc::tc_fence_after();
        const uint32_t sa = smem_base + stage * stage_bytes;
        const uint32_t sb = sa + a_bytes;
        uint32_t d_tmem = tmem_base;
        bool first = kb == 0;
        if (MODE == GATE) {
          const int g = kb / p.kb_per_group;
          d_tmem = tmem_base + g * p.Ep;
          first = (kb % p.kb_per_group) == 0;
        }
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = MODE == DWG ? tc::smem_desc_sw128(sa + k * 2048, 8192, 1024)
                                          : tc::smem_desc_sw128(sa + k * 32, 16, 1024);
          const uint64_t bd = MODE == DWG ? tc::smem_desc_sw128(sb + k * 2048, 8192, 1024)
                                          : tc::smem_desc_sw128(sb + k * 32, 16, 1024);
          tc::mma_bf16(d_tmem, ad, bd, idesc, (!first || k) ? 1u : 0u);
        }
        tc::mma_commit(&empty_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      tc::mma_commit(done_bar);
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int sub = warp & 3;
    const int row = sub * 32 + lane;                 // accumulator row = TMEM lane
    const uint32_t t_row = tmem_base + ((uint32_t)(sub * 32) << 16);
    if (nkb > 0) {
      tc::mbar_wait(done_bar, 0);
      tc::tc_fence_after();
    }
    if (MODE == GATE) {
      // The operand ring is idle once done_bar fired: reuse it for the logits / probs block
      // ls [128][E+1], the uniform-noise block us [128][E+1] and the decisions ss [128][E+1].
      const int LP = p.E + 1;
      float* ls = s_misc;                              // [128][E+1] logits
      // ---- logits: TwoSum over the NG K-group accumulators
      for (int c0 = 0; c0 < p.Ep; c0 += 16) {
        float sacc[16], cacc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) sacc[j] = cacc[j] = 0.f;
        for (int g = 0; g < p.ng; ++g) {
          uint32_t r[16];
          tc::tmem_ld16(t_row + g * p.Ep + c0, r);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float v = __uint_as_float(r[j]);
            const float s1 = sacc[j] + v;
            const float bp = s1 - sacc[j];
            cacc[j] += (sacc[j] - (s1 - bp)) + (v - bp);
            sacc[j] = s1;
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < p.E) ls[row * LP + c0 + j] = sacc[j] + cacc[j];
      }
      // ---- coalesced store of the fp32 logits block (steps 2-3 run in gate_softmax_tpt_kernel)
      tc::tc_fence_before();
      named_bar_sync(1, 128);
      const int et = threadIdx.x - 64;
      const int ntok = min(128, p.T - m0);
      for (int i = et; i < ntok * p.E; i += 128) p.logits[(long long)m0 * p.E + i] = ls[(i / p.E) * LP + (i % p.E)];
    } else {
      // ---- dW_g partial [split][d][E] = acc[:, e] (hi part) + acc[:, Ep + e] (lo part)
      const int m = m0 + row;
      float* dst = p.part + ((long long)blockIdx.y * p.d + m) * p.E;
      for (int c0 = 0; c0 < p.Ep; c0 += 16) {
        uint32_t rh[16], rl[16];
        tc::tmem_ld16(t_row + c0, rh);
        tc::tmem_ld16(t_row + p.Ep + c0, rl);
        tc::tmem_ld_wait();
        if (m >= p.d) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c0 + j < p.E) dst[c0 + j] = nkb > 0 ? __uint_as_float(rh[j]) + __uint_as_float(rl[j]) : 0.f;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ---------------------------------------------------------------- fused persistent gate
// Steps 1-3 in one persistent kernel (E % 16 == 0, E <= 64): x tiles stream through a 4-stage
// TMA ring, logits accumulate in NG K-group TMEM column blocks (the same grouping and TwoSum as
// the GATE epilogue above), two TMEM accumulators let tile i+1's loads and MMAs overlap tile i's
// epilogue.  Epilogue: 4 TMEM warps (thread = token row) add the K groups and write the fp32
// logits block to a double-buffered shared [128][E+1] buffer; 16 softmax warps then give each
// token 4 adjacent lanes (E/4 experts each): Gumbel noise, tau-softmax (max / sum combined over
// the 4 lanes by xor shuffles), threshold / guard / top-1 decision and band test as in
// gate_softmax_tpt_kernel, u read and probs / slot written as 256-byte row segments.
// Near-boundary tokens are queued for gate_refine_kernel (fp64), as before.  The logits never
// reach HBM.
#ifndef MOE_FG_STAGES
#define MOE_FG_STAGES 4
#endif
constexpr int FG_STAGES = MOE_FG_STAGES;   // x-tile ring depth (24 KB stages at E = 64)
constexpr int FG_SWARPS = 16;                     // 512 threads = 128 tokens x 4 lanes
constexpr int FG_THREADS = 64 + 128 + 32 * FG_SWARPS;

struct FgParams {
  int T, d, E, ng, kb_per_group, nkb, ntiles, nblk;
  float tau, thr;
  int top1;
  const float* u;
  float* probs;
  int* slot;
  int* counts;
  int* blk_cnt;
  int* near_band;
  int* flags;
  int* rq_count;
  int* rq_list;
};

// merge two (best, second, argmax) triples; ties keep the lower expert index as best
__device__ __forceinline__ void top2_merge(float& b, float& s, int& a, float b2, float s2, int a2) {
  if (b2 > b || (b2 == b && a2 < a)) {
    s = fmaxf(b, s2);
    b = b2;
    a = a2;
  } else {
    s = fmaxf(s, b2);
  }
}

template <int E_T>
__global__ void __launch_bounds__(FG_THREADS, 1)
    gate_fused_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, FgParams p) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = ((E_T * BK * 2) + 1023) & ~1023;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int LP = E_T + 4;                      // row pitch of the logits block (16-byte aligned rows)
  constexpr int EPT = E_T / 4;                     // experts per lane
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_u32 & 1023)) & 1023);
  float* lbuf = reinterpret_cast<float*>(smem + FG_STAGES * STAGE);      // [2][128][LP]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(lbuf + 2 * 128 * LP);
  uint64_t* empty_bar = full_bar + FG_STAGES;
  uint64_t* tfull_bar = empty_bar + FG_STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* lfull_bar = tempty_bar + 2;
  uint64_t* lempty_bar = lfull_bar + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(lempty_bar + 2);
  int* s_cnt0 = reinterpret_cast<int*>(s_tmem + 4);     // [2][E_T] per-tile counts (double-buffered by tile parity)
  int* s_band0 = s_cnt0 + 2 * E_T;                        // [2]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmX);
    tc::tma_prefetch(&tmW);
    for (int i = 0; i < FG_STAGES; ++i) {
      tc::mbar_init(&full_bar[i], 1);
      tc::mbar_init(&empty_bar[i], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull_bar[a], 1);
      tc::mbar_init(&tempty_bar[a], 4);
      tc::mbar_init(&lfull_bar[a], 4);
      tc::mbar_init(&lempty_bar[a], FG_SWARPS);
    }
    tc::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 2 * E_T; i += FG_THREADS) s_cnt0[i] = 0;
  if (threadIdx.x < 2) s_band0[threadIdx.x] = 0;
  if (warp == 1) tc::tmem_alloc(s_tmem, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const int m0 = tile * BM;
        for (int kb = 0; kb < p.nkb; ++kb) {
          tc::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE;
          tc::mbar_arrive_expect_tx(&full_bar[stage], A_BYTES + E_T * BK * 2);
          tc::tma_load_2d(sa, &tmX, &full_bar[stage], kb * BK, m0);
          tc::tma_load_2d(sa + A_BYTES, &tmW, &full_bar[stage], kb * BK, 0);
          if (++stage == FG_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(BM, E_T, 0, 0);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      const uint32_t smem_base = tc::smem_u32(smem);
      for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        tc::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        for (int kb = 0; kb < p.nkb; ++kb) {
          tc::mbar_wait(&full_bar[stage], phase);
          tc::tc_fence_after();
          const uint32_t sa = smem_base + stage * STAGE;
          const uint32_t sb = sa + A_BYTES;
          const int g = kb / p.kb_per_group;
          const bool first = (kb % p.kb_per_group) == 0;
          const uint32_t d_tmem = tmem_base + acc * 256 + g * E_T;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc::mma_bf16(d_tmem, tc::smem_desc_sw128(sa + k * 32, 16, 1024), tc::smem_desc_sw128(sb + k * 32, 16, 1024),
                         idesc, (!first || k) ? 1u : 0u);
          tc::mma_commit(&empty_bar[stage]);
          if (++stage == FG_STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ TMEM warps: logits block
    const int row = (warp & 3) * 32 + lane;
    const uint32_t t_row = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    int acc = 0, it = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
      const int b = it & 1;
      tc::mbar_wait(&tfull_bar[acc], acc_phase);
      tc::tc_fence_after();
      tc::mbar_wait(&lempty_bar[b], ((it >> 1) & 1) ^ 1);
      float* L = lbuf + (b * 128 + row) * LP;
#pragma unroll
      for (int c0 = 0; c0 < E_T; c0 += 16) {
        float sacc[16], cacc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) sacc[j] = cacc[j] = 0.f;
        for (int g = 0; g < p.ng; ++g) {
          uint32_t r[16];
          tc::tmem_ld16(t_row + acc * 256 + g * E_T + c0, r);
          tc::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float v = __uint_as_float(r[j]);
            const float s1 = sacc[j] + v;
            const float bp = s1 - sacc[j];
            cacc[j] += (sacc[j] - (s1 - bp)) + (v - bp);
            sacc[j] = s1;
          }
        }
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(L + c0 + j) = make_float4(sacc[j] + cacc[j], sacc[j + 1] + cacc[j + 1],
                                                               sacc[j + 2] + cacc[j + 2], sacc[j + 3] + cacc[j + 3]);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(&tempty_bar[acc]);
        tc::mbar_arrive(&lfull_bar[b]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ------------------------------------------------------------ softmax lanes: steps 2-3
    const int st = threadIdx.x - 192;                  // 0..511
    const int tok = st >> 2, q = st & 3;               // token of the tile, quarter of its experts
    const int e0 = q * EPT;
    // the softmax runs in base 2: z2 = (L + zeta) log2(e) / tau, p = 2^(z2 - max z2) (one multiply
    // and one ex2.approx per entry instead of a division and an expf; the arithmetic per entry,
    // two logf included, is about the time of the entry's HBM stream at C4)
    const float s2 = 1.4426950408889634f / p.tau;
    int it = 0;
    for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++it) {
      const int b = it & 1;
      const int t = tile * BM + tok;
      const bool live = t < p.T;
      int* s_cnt = s_cnt0 + b * E_T;
      int* s_band = s_band0 + b;
      // the noise row segment is fetched before waiting for the logits
      float U[EPT];
      if (p.u && live) {
#pragma unroll
        for (int j = 0; j < EPT; j += 4) {
          const float4 w = ld_nc_f4(p.u + (long long)t * p.E + e0 + j);
          U[j] = w.x; U[j + 1] = w.y; U[j + 2] = w.z; U[j + 3] = w.w;
        }
      }
      tc::mbar_wait(&lfull_bar[b], (it >> 1) & 1);
      float Z[EPT];
      const float* L = lbuf + (b * 128 + tok) * LP + e0;
#pragma unroll
      for (int j = 0; j < EPT; j += 4) {
        const float4 w = *reinterpret_cast<const float4*>(L + j);
        Z[j] = w.x; Z[j + 1] = w.y; Z[j + 2] = w.z; Z[j + 3] = w.w;
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&lempty_bar[b]);
      // ---- noise, tau-softmax
      float mx = -INFINITY;
      bool bad = false;
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        if (!isfinite(Z[j])) bad = true;
        const float zeta = p.u ? -logf(-logf(U[j])) : 0.f;
        Z[j] = (Z[j] + zeta) * s2;
        mx = fmaxf(mx, Z[j]);
      }
      if (bad && live && atomicOr(&p.flags[0], kFlagNonFinite) == 0) p.flags[1] = t;
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        Z[j] = ex2_approx(Z[j] - mx);
        sum += Z[j];
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      const float inv = 1.0f / sum;
      bool any_pass = false, near = false, band_thr = false;
      float best = -1.f, second = -1.f;
      int am = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const float pe = Z[j] * inv;
        Z[j] = pe;
        if (pe > p.thr) any_pass = true;
        const float dt = fabsf(pe - p.thr);
        if (dt < kRefine) near = true;
        if (dt < kBand) band_thr = true;
        if (pe > best) { second = best; best = pe; am = e0 + j; }
        else if (pe > second) second = pe;
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        any_pass |= __shfl_xor_sync(0xffffffffu, (int)any_pass, o) != 0;
        near |= __shfl_xor_sync(0xffffffffu, (int)near, o) != 0;
        band_thr |= __shfl_xor_sync(0xffffffffu, (int)band_thr, o) != 0;
        const float b2 = __shfl_xor_sync(0xffffffffu, best, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, second, o);
        const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
        top2_merge(best, second, am, b2, s2, a2);
      }
      const bool argmax_decided = p.top1 || !any_pass;
      if (p.top1) near = false;
      if (argmax_decided && best - second < kRefine) near = true;
      uint32_t sv[EPT];
      if (near) {
        if (live && q == 0) p.rq_list[atomicAdd(p.rq_count, 1)] = t;   // decided (and counted) by gate_refine_kernel
#pragma unroll
        for (int j = 0; j < EPT; ++j) sv[j] = 0xffffffffu;
      } else {
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
          const bool sel = argmax_decided ? (e0 + j == am) : (Z[j] > p.thr);
          sv[j] = sel ? 0u : 0xffffffffu;
          if (sel && live) atomicAdd(&s_cnt[e0 + j], 1);
        }
        const bool in_band = argmax_decided ? (best - second) < kBand : band_thr;
        if (in_band && live && q == 0) atomicAdd(s_band, 1);
      }
      if (live) {
#pragma unroll
        for (int j = 0; j < EPT; j += 4) {
          *reinterpret_cast<float4*>(p.probs + (long long)t * p.E + e0 + j) = make_float4(Z[j], Z[j + 1], Z[j + 2], Z[j + 3]);
          *reinterpret_cast<uint4*>(p.slot + (long long)t * p.E + e0 + j) = make_uint4(sv[j], sv[j + 1], sv[j + 2], sv[j + 3]);
        }
      }
      named_bar_sync(2, 32 * FG_SWARPS);
      for (int e = st; e < p.E; e += 32 * FG_SWARPS) {
        const int c = s_cnt[e];
        p.blk_cnt[(long long)e * p.nblk + tile] = c;
        if (c) atomicAdd(&p.counts[e], c);
        s_cnt[e] = 0;
      }
      if (st == 0 && s_band[0]) {
        atomicAdd(p.near_band, s_band[0]);
        s_band[0] = 0;
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, 512);
  }
}

// fp64 decisions for the deferred tokens (block per token)
constexpr int kRefineThreads = 1024;   // 4x the k slices of 256 threads: C4 refine 22.3 -> 19.6 us, C3 10.7 -> 9.8 us
__global__ void __launch_bounds__(kRefineThreads) gate_refine_kernel(const bf16* __restrict__ x, const bf16* __restrict__ Wg,
                                                          const float* __restrict__ u, int d, int E, float tau, float thr,
                                                          int top1, float* __restrict__ probs, int* __restrict__ slot,
                                                          int* __restrict__ counts, int* __restrict__ blk_cnt, int nblk,
                                                          int* __restrict__ near_band, const int* __restrict__ rq_count,
                                                          const int* __restrict__ rq_list) {
  __shared__ RefineSmem sm;
  const int n = *rq_count;
  for (int q = blockIdx.x; q < n; q += gridDim.x)
    gate_token_refine_block<bf16, kRefineThreads>(rq_list[q], x, Wg, u, d, E, tau, thr, top1, probs, slot, counts, blk_cnt, nblk, BM,
                                  near_band, sm);
}

// ------------------------------------------------------------------ small layout kernels
// WgT [Ep, d] bf16 (rows >= E zero) from W_g [d, E]; block 0 also zeroes the step's counters
// (counts [E], near_band, the refine queue length): no memset nodes before the gate kernel
__global__ void wg_transpose_kernel(const bf16* __restrict__ Wg, int d, int E, int Ep, bf16* __restrict__ WgT,
                                    int* __restrict__ counts, int* __restrict__ near_band, int* __restrict__ rq_count) {
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < E; i += blockDim.x) counts[i] = 0;
    if (threadIdx.x == 0) { *near_band = 0; *rq_count = 0; }
  }
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)Ep * d) return;
  const int e = (int)(i / d), k = (int)(i % d);
  WgT[i] = e < E ? Wg[(long long)k * E + e] : __float2bfloat16_rn(0.f);
}
// Wg2 [d, Kp] = [W_g | W_g | 0]  (B operand of the dense dL W_g^T GEMM with the hi | lo split of dL)
__global__ void wg_double_kernel(const bf16* __restrict__ Wg, int d, int E, int Ep, int Kp, bf16* __restrict__ Wg2) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)d * Kp) return;
  const int n = (int)(i / Kp), k = (int)(i % Kp);
  const int e = k < Ep ? k : k - Ep;
  Wg2[i] = (k < 2 * Ep && e < E) ? Wg[(long long)n * E + e] : __float2bfloat16_rn(0.f);
}
// dL2 [T, Kp] = [hi(dL) | lo(dL) | 0], hi = bf16(dL), lo = bf16(dL - hi); thread = 8 columns (16 B)
__global__ void dl_split_kernel(const float* __restrict__ dL, int T_, int E, int Ep, int Kp, bf16* __restrict__ dL2) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;     // vector index
  const int vpr = Kp / 8;
  if (i >= (long long)T_ * vpr) return;
  const long long t = i / vpr;
  const int k0 = (int)(i % vpr) * 8;
  const float* row = dL + t * E;
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int k = k0 + j;
    float o = 0.f;
    if (k < Ep) {
      if (k < E) o = __bfloat162float(__float2bfloat16_rn(row[k]));
    } else if (k < 2 * Ep && k - Ep < E) {
      const float f = row[k - Ep];
      o = f - __bfloat162float(__float2bfloat16_rn(f));
    }
    v[j] = o;
  }
  st_v4(dL2 + t * Kp + k0, pack16(v, bf16()));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode() {
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
static bool map2d(CUtensorMap* m, const void* ptr, long long rows, long long cols, int box_cols, int box_rows) {
  EncodeTiledFn f = encode();
  if (!f || !ptr) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int E_T>
static cudaError_t launch_fused(const CUtensorMap& mX, const CUtensorMap& mW, const FgParams& p, int grid,
                                cudaStream_t s) {
  constexpr int STAGE = BM * BK * 2 + (((E_T * BK * 2) + 1023) & ~1023);
  size_t smem = 1024 + FG_STAGES * STAGE + 2 * 128 * (E_T + 4) * 4 + 1024;
  if (smem < 120 * 1024) smem = 120 * 1024;      // one CTA per SM (each allocates all 512 TMEM columns)
  auto k = gate_fused_tc_kernel<E_T>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, FG_THREADS, smem, s>>>(mX, mW, p), count_launch();
  return cudaGetLastError();
}

static bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] && v[0] != '0';
}

static int pow2_cols(int c) {
  int p = 32;
  while (p < c) p <<= 1;
  return p;
}

template <int MODE>
static cudaError_t launch(const CUtensorMap& a, const CUtensorMap& b, const Params& p, dim3 grid, int bn,
                          size_t misc_bytes, cudaStream_t s) {
  const int stage_bytes = BM * BK * 2 + ((bn * BK * 2 + 1023) & ~1023);
  const size_t smem = 1024 + Stages<MODE>::N * stage_bytes + 1024 + misc_bytes;
  auto k = gate_tc_kernel<MODE>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<grid, Threads<MODE>::N, smem, s>>>(a, b, p), count_launch();
  return cudaGetLastError();
}

static cudaError_t launch_dl_split(const float* dL, int T, int E, int Ep, int Kp, bf16* dL2, cudaStream_t s) {
  const long long n = (long long)T * (Kp / 8);
  if (n == 0) return cudaSuccess;
  dl_split_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dL, T, E, Ep, Kp, dL2), count_launch();
  return cudaGetLastError();
}

}  // namespace tcgate

// E <= 64: the GATE epilogue parks the [128][E+1] noise block in the (2-stage) operand ring
bool gate_tc_supported(const moe_ctx* c) { return c->dtype == 1 && c->use_tc && c->E <= 64 && c->d % 64 == 0; }

static int gate_Ep(int E) { return (E + 15) / 16 * 16; }
static int gate_Kp(int E) { return (2 * gate_Ep(E) + 63) / 64 * 64; }

cudaError_t gate_tc_forward(const moe_ctx* c, const void* x, const void* Wg, const float* u, float tau, float thr,
                            int top1, float* probs, int32_t* slot, int32_t* counts, int32_t* near_band,
                            cudaStream_t s) {
  using namespace tcgate;
  const int E = c->E, d = c->d, Ep = gate_Ep(E);
  bf16* WgT = reinterpret_cast<bf16*>(c->gate_scratch);
  wg_transpose_kernel<<<(unsigned)(((long long)Ep * d + 255) / 256), 256, 0, s>>>((const bf16*)Wg, d, E, Ep, WgT,
                                                                                  counts, near_band, c->rq),
      count_launch();
  CUtensorMap mA, mB;
  if (!map2d(&mA, x, c->T, d, 64, BM) || !map2d(&mB, WgT, Ep, d, 64, Ep)) return cudaErrorInvalidValue;
  Params p{};
  p.mode = GATE; p.T = c->T; p.d = d; p.E = E; p.Ep = Ep;
  const int nkb = d / BK;
  int ng = 256 / Ep;                      // <= 256 TMEM columns per accumulator
  if (ng > nkb) ng = nkb;
  p.kb_per_group = (nkb + ng - 1) / ng;
  p.ng = (nkb + p.kb_per_group - 1) / p.kb_per_group;
  p.tmem_cols = pow2_cols(p.ng * Ep);
  p.logits = c->logits;
  cudaError_t e = cudaSuccess;
  const bool fused = E % 16 == 0 && c->T > 0 && !getenv_flag("MOE_GATE_UNFUSED");
  if (fused) {
    // steps 1-3 in one persistent kernel (logits stay on chip; near tokens refined inline)
    FgParams q{};
    q.T = c->T; q.d = d; q.E = E; q.ng = p.ng; q.kb_per_group = p.kb_per_group; q.nkb = nkb;
    q.ntiles = c->nblk; q.nblk = c->nblk; q.tau = tau; q.thr = thr; q.top1 = top1;
    q.u = u; q.probs = probs; q.slot = slot;
    q.counts = counts; q.blk_cnt = c->blk_cnt; q.near_band = near_band; q.flags = c->flags;
    q.rq_count = c->rq; q.rq_list = c->rq + 1;
    const int grid = c->nblk < c->sm_count ? c->nblk : c->sm_count;
    switch (E) {
      case 16: e = launch_fused<16>(mA, mB, q, grid, s); break;
      case 32: e = launch_fused<32>(mA, mB, q, grid, s); break;
      case 48: e = launch_fused<48>(mA, mB, q, grid, s); break;
      default: e = launch_fused<64>(mA, mB, q, grid, s); break;
    }
    if (e != cudaSuccess) return e;
  } else {
    const size_t misc = sizeof(int) * 132 + sizeof(float) * 128 * (E + 1);
    if ((e = launch<GATE>(mA, mB, p, dim3(c->nblk), Ep, misc, s)) != cudaSuccess) return e;
    if ((e = launch_gate_softmax_tpt(c, c->logits, u, tau, thr, top1, probs, slot, counts, near_band, s)) !=
        cudaSuccess)
      return e;
  }
  gate_refine_kernel<<<c->sm_count, kRefineThreads, 0, s>>>((const bf16*)x, (const bf16*)Wg, u, d, E, tau, thr, top1, probs, slot,
                                                 counts, c->blk_cnt, c->nblk, near_band, c->rq, c->rq + 1),
      count_launch();
  return cudaGetLastError();
}

// dxg [T, d] bf16 = dlogits W_g^T on the persistent CTA-pair GEMM (dL as a hi | lo bf16 pair:
// A = [hi | lo] [T, Kp], B = [W_g | W_g] [d, Kp]); moe_dispatch_bwd adds it in its gather pass.
void* gate_dl2_buffer(const moe_ctx* c) {
  return reinterpret_cast<bf16*>(c->gate_scratch) + (size_t)c->d * gate_Kp(c->E);
}

cudaError_t gate_tc_dx(const moe_ctx* c, const float* dlogits, const void* Wg, void* dx_bf16, bool have_split,
                       cudaStream_t s) {
  using namespace tcgate;
  const int E = c->E, d = c->d, Ep = gate_Ep(E), Kp = gate_Kp(E), T = c->T;
  bf16* Wg2 = reinterpret_cast<bf16*>(c->gate_scratch);
  bf16* dL2 = Wg2 + (size_t)d * Kp;
  wg_double_kernel<<<(unsigned)(((long long)d * Kp + 255) / 256), 256, 0, s>>>((const bf16*)Wg, d, E, Ep, Kp, Wg2),
      count_launch();
  cudaError_t e = have_split ? cudaGetLastError() : launch_dl_split(dlogits, T, E, Ep, Kp, dL2, s);
  if (e != cudaSuccess) return e;
  return tc_dense_store(c, dL2, T, Kp, Wg2, d, dx_bf16, c->tok_off, s);
}

// dW_g = x^T dlogits  (split over T, deterministic reduction)
cudaError_t gate_tc_dwg(const moe_ctx* c, const void* x, const float* dlogits, float* dWg, bool have_split,
                        cudaStream_t s) {
  using namespace tcgate;
  const int E = c->E, d = c->d, Ep = gate_Ep(E), Kp = gate_Kp(E), T = c->T;
  bf16* Wg2 = reinterpret_cast<bf16*>(c->gate_scratch);
  bf16* dL2 = Wg2 + (size_t)d * Kp;
  cudaError_t e0 = have_split ? cudaSuccess : launch_dl_split(dlogits, T, E, Ep, Kp, dL2, s);
  if (e0 != cudaSuccess) return e0;
  CUtensorMap mA, mB;
  if (!map2d(&mA, x, T, d, 64, 64) || !map2d(&mB, dL2, T, Kp, 64, 64)) return cudaErrorInvalidValue;
  const int m_tiles = (d + BM - 1) / BM;
  // one CTA per SM (measured: 2 per SM / fixed 16 or 32 splits are 5-45% slower at C2, C4, C5)
  int splits = c->sm_count / m_tiles;
  if (splits < 1) splits = 1;
  if (splits > c->dwg_splits_max) splits = c->dwg_splits_max;
  int split_rows = ((T + splits - 1) / splits + BK - 1) / BK * BK;
  splits = (T + split_rows - 1) / split_rows;
  if (splits < 1) splits = 1;
  Params p{};
  p.mode = DWG; p.T = T; p.d = d; p.E = E; p.Ep = Ep; p.Kp = Kp; p.split_rows = split_rows;
  p.tmem_cols = pow2_cols(Kp);
  p.part = c->part;
  cudaError_t e = launch<DWG>(mA, mB, p, dim3(m_tiles, splits), Kp, 0, s);
  if (e != cudaSuccess) return e;
  return launch_reduce_splits(c->part, splits, (long long)d * E, dWg, s);
}

}  // namespace moe
