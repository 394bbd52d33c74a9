// gemm_tc.cu -- persistent, warp-specialised tcgen05 grouped GEMM for the expert FFN
// (step 5 and B5), run as CTA PAIRS (cluster of 2, tcgen05 cta_group::2).
//
// One pair computes a 256 x 256 fp32 tile: each CTA holds 128 rows of A and 128 rows
// (N-columns) of B per 64-deep K stage (32 KB / stage / CTA), the pair leader issues
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16) and each CTA's TMEM receives its own
// 128 accumulator rows.  Two 256-column TMEM accumulators let the epilogue of tile i
// overlap the mainloop of tile i+1.  Operands arrive by TMA (128-byte swizzle) into a
// 5-7 stage ring; the epilogue (4 x EpiCfg::PER_Q warps, thread = accumulator row)
// reads TMEM with tcgen05.ld, applies the fused bias / GELU / GELU' / fp32 variants and
// writes bf16 results through shared memory with TMA bulk-tensor stores.  The GELU'
// operand a is TMA-loaded into the same staging buffers two chunks ahead.
//
// Roles (64 + 128 x PER_Q threads / CTA): warp 0 = TMA producer, warp 1 = TMEM allocator +
//   MMA issuer (leader CTA only), warps 2.. = epilogue.
// Scheduling (static, per pair): ROWS mode (ragged M): a tile is a pair of 128-row blocks
//   of ONE expert (segments are 128-aligned) x one 256-wide N block; the expert comes from
//   the device offsets[].  An expert's odd last block is a HALF tile: an M = 128 pair MMA
//   (64 rows per CTA), whose accumulator holds rows 0-63 x columns 0-127 in TMEM lanes 0-63
//   and the same rows x columns 128-255 in lanes 64-127 -- no CTA computes pad rows.
//   KGRP mode (ragged K, weight gradients): tiles = G x ceil(M/256) x ceil(N/256), K range
//   of group g = [offsets[g], offsets[g+1]); empty groups store zeros.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>

#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"

namespace moe {

namespace {

constexpr int BM = 128;                      // rows per CTA (pair tile: 256)
constexpr int BN = 256;                      // pair tile width; each CTA stages BNH rows of B
constexpr int BNH = 128;
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;         // 16 KB
constexpr int B_BYTES = BNH * BK * 2;        // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;               // 2 accumulators x 256 fp32 columns
constexpr int CHUNKS = 256 / 32;
constexpr int CHUNK_BYTES = 32 * 32 * 2;     // one 32x32 bf16 sub-tile (TMA box, 64-byte swizzle)
constexpr int MAX_G = 128;
constexpr int SMEM_LIMIT = 232448;

// TEPI_BIAS_GELU writes (GELU'(a), GELU(a)); TEPI_BIAS_GELU_H writes GELU(a) only (recompute mode)
enum TcEpi { TEPI_BIAS_GELU = 0, TEPI_BIAS = 1, TEPI_GELU_BWD = 2, TEPI_STORE = 3, TEPI_F32 = 4, TEPI_BIAS_GELU_H = 5 };

// Epilogue warps per TMEM lane quarter, per epilogue kind (measured at C2, C4 and C5 steps
// 5 / 19, profiles/r01/s2/epi_warps.txt): the GELU epilogues need 3 (ALU + staging work per
// chunk; 2 is 2% faster for GEMM1 at d >= 768 but 5% slower at d = 512), bias / store run
// best with 2 and the long-K fp32 weight gradients with 1 (fewer warps contending for shared
// memory, and a smaller staging area leaves room for more operand stages).
#ifndef MOE_EPQ_GELU
#define MOE_EPQ_GELU 3
#endif
#ifndef MOE_EPQ_BIAS
#define MOE_EPQ_BIAS 2
#endif
#ifndef MOE_EPQ_GBWD
#define MOE_EPQ_GBWD 3
#endif
#ifndef MOE_EPQ_STORE
#define MOE_EPQ_STORE 2
#endif
#ifndef MOE_EPQ_F32
#define MOE_EPQ_F32 1
#endif
// (GELU and fp32 weight-gradient epilogues: 1 buffer per warp -- the smaller staging area buys
// operand stages, C4 GEMM1 -1.7%, weight gradients -2%; bias / store keep 2, profiles/r01/s2/epi_warps.txt)
// GELU' operand ring of the dgrad2 epilogue: MOE_NB_GBWD staging buffers per warp, the operand of
// chunk seq + MOE_AUXD loaded while chunk seq is processed (MOE_NB_GBWD - MOE_AUXD stores in flight)
#ifndef MOE_NB_GBWD
#define MOE_NB_GBWD 4
#endif
#ifndef MOE_AUXD
#define MOE_AUXD 2
#endif
#ifndef MOE_NB_GELU
#define MOE_NB_GELU 1
#endif
#ifndef MOE_NB_BIAS
#define MOE_NB_BIAS 2
#endif
#ifndef MOE_NB_STORE
#define MOE_NB_STORE 2
#endif
#ifndef MOE_NB_F32
#define MOE_NB_F32 1
#endif
template <int EPI, int QOV = 0> struct EpiCfg {   // QOV: epilogue warps per quarter override (0 = the kind's default)
  // thread = accumulator row; epilogue warp (quarter q, part j) owns chunks j, j + PER_Q, ... of the 8 x 32 columns
  static constexpr int PER_Q = QOV ? QOV : EPI == TEPI_BIAS_GELU || EPI == TEPI_BIAS_GELU_H ? MOE_EPQ_GELU
                               : EPI == TEPI_BIAS ? MOE_EPQ_BIAS
                               : EPI == TEPI_GELU_BWD ? MOE_EPQ_GBWD
                               : EPI == TEPI_STORE ? MOE_EPQ_STORE : MOE_EPQ_F32;
  static constexpr int WARPS = 4 * PER_Q;
  static constexpr int THREADS = 64 + 32 * WARPS;
  static constexpr int NOUT = EPI == TEPI_BIAS_GELU ? 2 : (EPI == TEPI_F32 ? 0 : 1);  // bf16 TMA-stored outputs
  // staging buffers per warp (GELU' bwd: 4, its a-operand loads run two chunks ahead)
  static constexpr int NBUF = EPI == TEPI_GELU_BWD ? MOE_NB_GBWD
                              : EPI == TEPI_BIAS_GELU || EPI == TEPI_BIAS_GELU_H ? MOE_NB_GELU
                              : EPI == TEPI_BIAS ? MOE_NB_BIAS
                              : EPI == TEPI_STORE ? MOE_NB_STORE : MOE_NB_F32;
  // per-warp staging: NBUF chunk buffers of NOUT bf16 32x32 boxes, or of one fp32 32x32 box (F32)
  static constexpr int WARP_STAGE = EPI == TEPI_F32 ? NBUF * 2 * CHUNK_BYTES : NBUF * NOUT * CHUNK_BYTES;
  static constexpr int STAGING = WARPS * WARP_STAGE;
  static constexpr int BAR_BYTES = 2048;
  static constexpr int STAGES = (SMEM_LIMIT - 1024 - BAR_BYTES - STAGING) / STAGE_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + STAGING + 1024 + BAR_BYTES;
};

struct TcParams {
  int G;
  const int* offsets;     // [G+1]
  int M, N, K;            // ROWS: N, K used; KGRP: M, N used
  int rows_cap;           // ROWS: R_cap (rows of every row-layout buffer)
  int b_group_rows;       // ROWS: B tensor-map row offset of group g = g * b_group_rows
  float* out;             // KGRP fp32 output, row-major pitch ldo (+ g * out_g)
  long long ldo;
  long long out_g;
  const float* bias;      // fp32 copy (c->biasf), rows padded to 256 columns: + g * bias_g
  long long bias_g;
  bf16* o1;               // bf16 outputs (ROWS), pitch ldo_b -- used by the LSU store variant
  bf16* o2;
  long long ldo_b;
  float* colpart;         // TEPI_GELU_BWD: per-32-row column sums of da [R_cap/32][N] (bias gradient db1)
  int o12;                // GEMM1: gp and h are one [2][R_cap][f] buffer, stored with ONE 3D TMA op per chunk
  void* reserved1;        // (unused; keeps the parameter block's layout of the measured builds)
  int a3d, b3d;           // MN-major operand given as a 3D map {64, K rows, MN / 64}: one TMA op per stage
  // exchange / GEMM overlap (ROWS, peer-memory EP): before the first A load of an expert's tile the
  // producer waits until arrive[g] reaches arrive_target[g] (wrap-safe), then fences the async proxy
  const int* arrive;
  const int* arrive_target;
  int* flags;
};

// Acquire-poll of expert g's arrival counter (written by peers' ep2_copy_ordered_kernel with
// release adds).  Stops early when the plan raised MOE_ECAPACITY (dropped rows are counted anyway,
// but the step is re-run) and after a bounded spin (kFlagArrival instead of a hang).
__device__ __forceinline__ void wait_arrival(const TcParams& p, int g) {
  const int tgt = p.arrive_target[g];
  for (int spins = 0;; ++spins) {
    int v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p.arrive + g) : "memory");
    if ((int)((unsigned)v - (unsigned)tgt) >= 0) break;
    if (*reinterpret_cast<volatile int*>(p.flags) & kFlagCapacity) break;
    if (spins > (1 << 22)) {
      atomicOr(p.flags, kFlagArrival);
      break;
    }
    __nanosleep(256);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct Tile {
  int g, m_own, n0, kb0, nkb, row_end;
  int half;   // ROWS: the odd last 128-row block of an expert, run as an M = 128 pair MMA (64 rows per CTA)
};

template <bool KGRP>
__device__ __forceinline__ bool decode_tile(const TcParams& p, const int* s_off, const int* s_pair, int t,
                                            int n_tiles, uint32_t rank, Tile& tl) {
  if (!KGRP) {
    const int P = t / n_tiles, nt = t - P * n_tiles;
    int lo = 0, hi = p.G - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s_pair[mid] <= P) lo = mid; else hi = mid - 1;
    }
    tl.g = lo;
    const int pl = P - s_pair[lo];
    const int blocks = (s_off[lo + 1] - s_off[lo]) / BM;        // segments are 128-aligned
    tl.half = (blocks & 1) && 2 * pl + 1 == blocks;
    tl.m_own = s_off[lo] + 256 * pl + (tl.half ? 64 : 128) * (int)rank;
    tl.row_end = min(s_off[lo + 1], p.rows_cap);
    tl.n0 = nt * BN;
    tl.kb0 = 0;
    tl.nkb = (p.K + BK - 1) / BK;
  } else {
    const int m_tiles = (p.M + 255) / 256;
    const int per_g = m_tiles * n_tiles;
    tl.g = t / per_g;
    const int r = t - tl.g * per_g;
    const int mt = r / n_tiles, nt = r - mt * n_tiles;
    tl.m_own = mt * 256 + 128 * (int)rank;
    tl.half = 0;
    tl.row_end = p.M;
    tl.n0 = nt * BN;
    tl.kb0 = s_off[tl.g] / BK;
    tl.nkb = (s_off[tl.g + 1] - s_off[tl.g]) / BK;
  }
  return tl.nkb > 0;
}

template <int EPI, bool A_MN, bool B_MN, bool KGRP, int QOV = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(EpiCfg<EPI, QOV>::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO1, const __grid_constant__ CUtensorMap tmO2,
                   const __grid_constant__ CUtensorMap tmX, TcParams p) {
  using Cfg = EpiCfg<EPI, QOV>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int EPI_PER_Q = Cfg::PER_Q, EPI_WARPS = Cfg::WARPS, NUM_THREADS = Cfg::THREADS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = tc::smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024 - (raw_u32 & 1023)) & 1023);   // 1024-aligned (SWIZZLE_128B atoms)
  uint8_t* staging = smem + STAGES * STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + Cfg::STAGING);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* aux_bar = tempty_bar + 2;                               // [EPI_WARPS][8] (GELU' operand loads)
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(aux_bar + EPI_WARPS * 8);
  int* s_off = reinterpret_cast<int*>(s_tmem + 4);
  int* s_pair = s_off + (MAX_G + 1);

  const uint32_t rank = tc::cluster_rank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  for (int i = threadIdx.x; i <= p.G && i <= MAX_G; i += NUM_THREADS) s_off[i] = p.offsets[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int g = 0; g < p.G; ++g) {
      s_pair[g] = acc;
      acc += (s_off[g + 1] - s_off[g] + 255) / 256;
    }
    s_pair[p.G] = acc;
  }
  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
    if (Cfg::NOUT >= 1 || EPI == TEPI_F32) tc::tma_prefetch(&tmO1);
    if (Cfg::NOUT >= 2) tc::tma_prefetch(&tmO2);
    if (EPI == TEPI_GELU_BWD) tc::tma_prefetch(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full_bar[s], 1);
      tc::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull_bar[a], 1);
      tc::mbar_init(&tempty_bar[a], 2 * EPI_WARPS);
    }
    for (int i = 0; i < EPI_WARPS * 8; ++i) tc::mbar_init(&aux_bar[i], 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) {
    tc::tmem_alloc_pair(s_tmem, TMEM_COLS);
    tc::tmem_relinquish_pair();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem_base = *s_tmem;

  const int n_tiles = (p.N + BN - 1) / BN;
  const int total = KGRP ? p.G * ((p.M + 255) / 256) * n_tiles : s_pair[p.G] * n_tiles;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t smem_base = tc::smem_u32(smem);
      const uint32_t full_leader = tc::mapa(tc::smem_u32(full_bar), 0);
      int waited_g = -1;
      for (int t = cid; t < total; t += ncl) {
        Tile tl;
        if (!decode_tile<KGRP>(p, s_off, s_pair, t, n_tiles, rank, tl)) continue;
        if (!KGRP && p.arrive && tl.g != waited_g) {
          wait_arrival(p, tl.g);
          waited_g = tl.g;
        }
        const int n_own = tl.n0 + BNH * (int)rank;
        const int brow = KGRP ? 0 : tl.g * p.b_group_rows;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          tc::mbar_wait(&empty_bar[stage], phase ^ 1);
          if (leader) tc::mbar_arrive_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
          const uint32_t bar = full_leader + stage * 8;
          const uint32_t sa = smem_base + stage * STAGE_BYTES;
          const uint32_t sb = sa + A_BYTES;
          const int k = (tl.kb0 + kb) * BK;
          if (!A_MN) {
            tc::tma_load_2d_pair(sa, &tmA, bar, k, tl.m_own);
          } else if (p.a3d) {                      // both 64-wide MN chunks ([chunk][k][64]) in one op
            tc::tma_load_3d_pair(sa, &tmA, bar, 0, k, tl.m_own / 64);
          } else {
            tc::tma_load_2d_pair(sa, &tmA, bar, tl.m_own, k);
            tc::tma_load_2d_pair(sa + 8192, &tmA, bar, tl.m_own + 64, k);
          }
          if (!B_MN) {
            tc::tma_load_2d_pair(sb, &tmB, bar, k, brow + n_own);
          } else if (p.b3d) {
            tc::tma_load_3d_pair(sb, &tmB, bar, 0, brow + k, n_own / 64);
          } else {
            tc::tma_load_2d_pair(sb, &tmB, bar, n_own, brow + k);
            tc::tma_load_2d_pair(sb + 8192, &tmB, bar, n_own + 64, brow + k);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair leader)
    if (leader && lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(256, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      // half tiles: M = 128 across the pair (each CTA's first 64 A rows); the accumulator then holds
      // rows 0-63 x columns 0-127 in TMEM lanes 0-63 and the same rows x columns 128-255 in lanes
      // 64-127, columns 0-127 of the buffer (the 2-SM M = 128 data-path layout)
      constexpr uint32_t idesc_h = tc::idesc_bf16(128, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t smem_base = tc::smem_u32(smem);
      for (int t = cid; t < total; t += ncl) {
        Tile tl;
        if (!decode_tile<KGRP>(p, s_off, s_pair, t, n_tiles, rank, tl)) continue;
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
            // MN-major SW128: +2048 B per K=16 step, LBO = 8 KB (64-wide MN chunk), SBO = 1024
            const uint64_t ad = A_MN ? tc::smem_desc_sw128(sa + k * 2048, 8192, 1024)
                                     : tc::smem_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? tc::smem_desc_sw128(sb + k * 2048, 8192, 1024)
                                     : tc::smem_desc_sw128(sb + k * 32, 16, 1024);
            tc::mma_bf16_pair(d_tmem, ad, bd, tl.half ? idesc_h : idesc, (kb | k) != 0);
          }
          tc::mma_commit_pair_mc(tc::smem_u32(&empty_bar[stage]), 0x3);   // frees the slot in both CTAs
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit_pair_mc(tc::smem_u32(&tfull_bar[acc]), 0x3);       // accumulators ready in both CTAs
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9)
    const int ew = warp - 2;
    const int sub = warp & 3;                          // TMEM lane quarter this warp may access
    const int part = ew >> 2;                          // chunks part, part + 3, part + 6 (< 8) of the 8 x 32 columns
    const int nch = (CHUNKS - part + EPI_PER_Q - 1) / EPI_PER_Q;
    const int row_in_tile = sub * 32 + lane;
    const uint32_t stage_base = tc::smem_u32(staging) + ew * Cfg::WARP_STAGE;
    const uint32_t swz = (uint32_t)((lane >> 1) & 3);  // SWIZZLE_64B: 16-byte chunk q -> q ^ ((row >> 1) & 3)
    const uint32_t tempty_leader = tc::mapa(tc::smem_u32(tempty_bar), 0);
    const uint32_t auxb = tc::smem_u32(aux_bar + ew * 8);
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t seq = 0;                                   // this warp's chunk sequence number (nch per tile)

    // this warp's rows / columns / chunk count in a tile: full tiles -> rows sub*32.., all 8 chunks
    // of 32 columns shared by the quarter's warps; half tiles -> rows (sub&1)*32.. of the CTA's 64,
    // column half (sub>>1)*128, 4 chunks
    auto rows0 = [&](const Tile& x) { return x.half ? (sub & 1) * 32 : sub * 32; };
    auto cols0 = [&](const Tile& x) { return x.half ? (sub >> 1) * 128 : 0; };
    auto nchunks = [&](const Tile& x) { return x.half ? (CHUNKS / 2 - part + EPI_PER_Q - 1) / EPI_PER_Q : nch; };

    // GELU' operand: TMA-load a[rows, 32 cols] MOE_AUXD chunks ahead into the staging buffers,
    // following the consumer's (tile, chunk) order with a cursor (the expert search runs once per
    // tile, not once per chunk: lane 0's chunk critical path)
    int aux_t = cid, aux_k = 0;
    uint32_t aux_seq = 0;
    bool aux_have = false;
    Tile tn{};
    auto aux_issue = [&]() {
      while (aux_t < total) {
        if (!aux_have) {
          decode_tile<KGRP>(p, s_off, s_pair, aux_t, n_tiles, rank, tn);
          aux_have = true;
        }
        if (aux_k < nchunks(tn)) {
          const int col = tn.n0 + cols0(tn) + (part + EPI_PER_Q * aux_k) * 32;
          const uint32_t b = aux_seq % Cfg::NBUF;
          tc::mbar_arrive_expect_tx_u32(auxb + b * 8, CHUNK_BYTES);
          tc::tma_load_2d_u32(stage_base + b * CHUNK_BYTES, &tmX, auxb + b * 8, col, tn.m_own + rows0(tn));
          ++aux_seq;
          ++aux_k;
          return;
        }
        aux_t += ncl;
        aux_k = 0;
        aux_have = false;
      }
    };
    if (EPI == TEPI_GELU_BWD && lane == 0) {
      for (int i = 0; i < MOE_AUXD; ++i) aux_issue();
    }

    for (int t = cid; t < total; t += ncl) {
      Tile tl;
      const bool nonempty = decode_tile<KGRP>(p, s_off, s_pair, t, n_tiles, rank, tl);
      const long long row = (long long)tl.m_own + row_in_tile;
      if (KGRP && !nonempty) {
        // empty expert -> zero gradient tile
        if (row < p.M) {
          float* o = p.out + (long long)tl.g * p.out_g + row * p.ldo;
          for (int k = 0; k < nch; ++k)
            for (int c = (part + EPI_PER_Q * k) * 32; c < (part + EPI_PER_Q * k) * 32 + 32; c += 4)
              if (tl.n0 + c < p.N) *reinterpret_cast<float4*>(o + tl.n0 + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        continue;
      }
      const int r0 = rows0(tl), coff = cols0(tl), nch_t = nchunks(tl);
      const bool warp_rows_ok = tl.m_own + r0 < tl.row_end;          // warp-uniform for ROWS tiles
      const float* bias_t = nullptr;                                 // padded fp32 bias row of this tile
      if (EPI == TEPI_BIAS_GELU || EPI == TEPI_BIAS || EPI == TEPI_BIAS_GELU_H)
        bias_t = p.bias + (long long)tl.g * p.bias_g + tl.n0 + coff;
      tc::mbar_wait_sleep(&tfull_bar[acc], acc_phase);
      tc::tc_fence_after();
      const uint32_t t_row = tmem_base + acc * BN + ((uint32_t)(sub * 32) << 16);
#pragma unroll 1
      for (int k = 0; k < nch_t; ++k, ++seq) {
        const int col = (part + EPI_PER_Q * k) * 32;     // TMEM column of the chunk
        const int n = tl.n0 + coff + col;                // output column
        uint32_t r[32];
        float4 bf[8];                                      // bias of this chunk (broadcast loads)
        if (EPI == TEPI_BIAS_GELU || EPI == TEPI_BIAS || EPI == TEPI_BIAS_GELU_H) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            bf[q] = ld_nc_f4(bias_t + col + 4 * q);
        }
        tc::tmem_ld32(t_row + col, r);
        tc::tmem_ld_wait();
        if (EPI == TEPI_F32) {
          // fp32 32x32 box (128-byte rows, SWIZZLE_128B) staged in smem, one TMA store: coalesced
          // full-line writes instead of 32 scattered 16-byte rows per store instruction
          const uint32_t fbuf = stage_base + (seq % Cfg::NBUF) * (2 * CHUNK_BYTES);
          if (seq >= (uint32_t)Cfg::NBUF) {
            if (lane == 0) tc::bulk_wait_read<Cfg::NBUF - 1>();
            __syncwarp();
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            tc::st_shared_v4(fbuf + lane * 128 + ((q ^ (lane & 7)) << 4),
                             make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]));
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            // M and N are multiples of 64: a 32x32 box is wholly inside the group's [M, N] block or outside
            if (tl.m_own + r0 < p.M && n < p.N)
              tc::tma_store_2d(&tmO1, fbuf, n, tl.g * p.M + tl.m_own + r0);
            tc::bulk_commit();
          }
          __syncwarp();
          continue;
        }
        const bool store = warp_rows_ok && n < p.N;
        const uint32_t buf = stage_base + (seq % Cfg::NBUF) * (Cfg::NOUT * CHUNK_BYTES);
        f32x2 v[16];                                       // packed fp32 pairs (FFMA2/FMUL2/FADD2)
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = f2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
        if (EPI == TEPI_GELU_BWD) {
          tc::mbar_wait_u32(auxb + (seq % Cfg::NBUF) * 8, (seq / Cfg::NBUF) & 1);
#pragma unroll
          for (int q = 0; q < 4; ++q) {                        // gp = GELU'(a) saved by the forward
            const uint4 g4 = tc::ld_shared_v4(buf + lane * 64 + ((q ^ swz) << 4));
            v[q * 4 + 0] = mul2(v[q * 4 + 0], bf16x2_to_f2(g4.x));   // da = dh (.) GELU'(a)
            v[q * 4 + 1] = mul2(v[q * 4 + 1], bf16x2_to_f2(g4.y));
            v[q * 4 + 2] = mul2(v[q * 4 + 2], bf16x2_to_f2(g4.z));
            v[q * 4 + 3] = mul2(v[q * 4 + 3], bf16x2_to_f2(g4.w));
          }
        } else {
          if (seq >= (uint32_t)Cfg::NBUF) {               // the group that last used this buffer must be read
            if (lane == 0) tc::bulk_wait_read<Cfg::NBUF - 1>();
            __syncwarp();
          }
          if (EPI == TEPI_BIAS_GELU || EPI == TEPI_BIAS || EPI == TEPI_BIAS_GELU_H) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              v[q * 2 + 0] = add2(v[q * 2 + 0], f2(bf[q].x, bf[q].y));
              v[q * 2 + 1] = add2(v[q * 2 + 1], f2(bf[q].z, bf[q].w));
            }
          }
        }
        if (EPI == TEPI_BIAS_GELU) {
          // out1 = GELU'(a) (kept for the backward), out2 = h = GELU(a): one Phi / exp per element
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t hw[4], gw[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              f32x2 h2, g2;
              gelu_and_prime_x2(v[q * 4 + j], h2, g2);
              hw[j] = f2_to_bf16x2(h2);
              gw[j] = f2_to_bf16x2(g2);
            }
            tc::st_shared_v4(buf + lane * 64 + ((q ^ swz) << 4), make_uint4(gw[0], gw[1], gw[2], gw[3]));
            tc::st_shared_v4(buf + CHUNK_BYTES + lane * 64 + ((q ^ swz) << 4), make_uint4(hw[0], hw[1], hw[2], hw[3]));
          }
        } else if (EPI == TEPI_BIAS_GELU_H) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t hw[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              f32x2 h2, g2;
              gelu_and_prime_x2(v[q * 4 + j], h2, g2, false);
              hw[j] = f2_to_bf16x2(h2);
            }
            tc::st_shared_v4(buf + lane * 64 + ((q ^ swz) << 4), make_uint4(hw[0], hw[1], hw[2], hw[3]));
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            tc::st_shared_v4(buf + lane * 64 + ((q ^ swz) << 4),
                             make_uint4(f2_to_bf16x2(v[q * 4]), f2_to_bf16x2(v[q * 4 + 1]), f2_to_bf16x2(v[q * 4 + 2]),
                                        f2_to_bf16x2(v[q * 4 + 3])));
        }
        tc::fence_proxy_async();
        __syncwarp();
        if (EPI == TEPI_GELU_BWD && p.colpart && store) {
          // db1 partial of this warp's 32 x 32 bf16 da sub-tile (fixed order): lane = (column pair
          // cp = lane & 15, row parity rp = lane >> 4) sums rows rp, rp+2, ..., then the two parities
          // are added.  Even/odd rows sit in opposite 64-byte bank halves: conflict-free.
          const uint32_t cp = lane & 15, rp = lane >> 4;
          f32x2 cs = f2(0.f);
#pragma unroll 8
          for (uint32_t i = 0; i < 16; ++i) {
            const uint32_t r = 2 * i + rp;
            const uint32_t addr = buf + r * 64 + (((cp >> 2) ^ ((r >> 1) & 3)) << 4) + (cp & 3) * 4;
            uint32_t w;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(addr));
            cs = add2(cs, bf16x2_to_f2(w));
          }
          float c0, c1;
          f2_split(cs, c0, c1);
          c0 += __shfl_xor_sync(0xffffffffu, c0, 16);
          c1 += __shfl_xor_sync(0xffffffffu, c1, 16);
          if (rp == 0)
            *reinterpret_cast<float2*>(p.colpart + (long long)((tl.m_own + r0) >> 5) * p.N + n + 2 * cp) =
                make_float2(c0, c1);
        }
        if (lane == 0) {
          if (store) {
            const int row0 = tl.m_own + r0;
            if (Cfg::NOUT == 2 && p.o12) {
              tc::tma_store_3d(&tmO1, buf, n, row0, 0);      // the [2][32][32] staging box: gp then h
            } else {
              tc::tma_store_2d(&tmO1, buf, n, row0);
              if (Cfg::NOUT == 2) tc::tma_store_2d(&tmO2, buf + CHUNK_BYTES, n, row0);
            }
          }
          tc::bulk_commit();                              // one (possibly empty) group per chunk
          if (EPI == TEPI_GELU_BWD) {
            // buffer (seq + AUXD) % NBUF was last stored at chunk seq + AUXD - NBUF
            tc::bulk_wait_read<MOE_NB_GBWD - MOE_AUXD>();
            aux_issue();
          }
        }
        __syncwarp();
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(tempty_leader + acc * 8);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if ((Cfg::NOUT > 0 || EPI == TEPI_F32) && lane == 0) tc::bulk_wait<0>();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  if (warp == 1) {
    __syncwarp();
    tc::tc_fence_after();
    tc::tmem_dealloc_pair(tmem_base, TMEM_COLS);
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
// box = {box_cols (inner), box_rows}; swizzle 128B for MMA operands (box_cols * 2 == 128),
// 64B for the 32x32 epilogue store boxes (box_cols * 2 == 64).
bool make_map(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long pitch, int box_cols,
              int box_rows, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn f = encode_fn();
  if (!f || !ptr) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
// MN-major operand as a 3D map {64 (MN, inner), rows (K), cols / 64 (MN chunk)}, box {64, 64, 2}:
// one TMA op fills the [chunk][k][64] stage layout of two 2D boxes.  Only when cols % 64 == 0
// (a partial last chunk would read past the row end instead of being zero-filled); returns
// false otherwise and the caller keeps the 2D map.
bool make_map_mn3d(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long pitch) {
  EncodeTiledFn f = encode_fn();
  if (!f || !ptr || cols % 64 != 0 || getenv("MOE_NO_MN3D")) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 2, 128};
  cuuint32_t box[3] = {64, 64, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// MN-major operand map: 3D when possible (flag set), else the 2D {64, 64} box map
bool make_map_mn(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long pitch, int& is3d) {
  is3d = make_map_mn3d(m, ptr, rows, cols, pitch) ? 1 : 0;
  return is3d || make_map(m, ptr, rows, cols, pitch, 64, 64);
}
bool make_store_map(CUtensorMap* m, const void* ptr, long long rows, long long cols) {
  return make_map(m, ptr, rows, cols, cols, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
}
// two [rows, cols] bf16 outputs, the second `gap` bytes after the first (gap >= rows*cols*2, a
// multiple of 16), as one 3D map with {32, 32, 2} boxes: the epilogue's two staged 32x32 boxes
// leave in one TMA op
bool make_store_map_pair(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long gap) {
  EncodeTiledFn f = encode_fn();
  if (!f || !ptr || gap < rows * cols * 2 || gap % 16 != 0 || gap >= (1ll << 40)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)gap};
  cuuint32_t box[3] = {32, 32, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// fp32 [rows, cols] row-major output, 32x32 boxes with 128-byte swizzled rows (weight gradients)
bool make_store_map_f32(CUtensorMap* m, const void* ptr, long long rows, long long cols) {
  EncodeTiledFn f = encode_fn();
  if (!f || !ptr) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int EPI, bool A_MN, bool B_MN, bool KGRP, int QOV = 0>
cudaError_t launch_tc(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& o1, const CUtensorMap& o2,
                      const CUtensorMap& x, const TcParams& p, long long tiles_upper, int sms, cudaStream_t s) {
  auto k = tc_gemm_kernel<EPI, A_MN, B_MN, KGRP, QOV>;
  constexpr int smem = EpiCfg<EPI, QOV>::SMEM;
  static_assert(smem <= SMEM_LIMIT, "shared memory budget");
  // the >48 KB shared-memory opt-in is per device: set it once for every device this
  // instantiation launches on (bit per device ordinal)
  static std::atomic<unsigned long long> attr_devs{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaGetLastError();
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_devs.load(std::memory_order_relaxed) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_devs.fetch_or(bit, std::memory_order_relaxed);
  }
  long long pairs = tiles_upper < sms / 2 ? tiles_upper : sms / 2;
  if (pairs <= 0) return cudaSuccess;
  k<<<(unsigned)(2 * pairs), EpiCfg<EPI, QOV>::THREADS, smem, s>>>(a, b, o1, o2, x, p), count_launch();
  return cudaGetLastError();
}

// fp32, 256-column-padded copies of b1 and b2 for the epilogues (one launch per forward):
// out = [El][fp] (b1, zero beyond f) then [El][dp] (b2, zero beyond d).
__global__ void bias_f32_kernel(const bf16* __restrict__ b1, const bf16* __restrict__ b2, int El, int f, int d,
                                int fp, int dp, float* __restrict__ out) {
  const long long n1 = (long long)El * fp, n = n1 + (b2 ? (long long)El * dp : 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float v = 0.f;
    if (i < n1) {
      const int g = (int)(i / fp), c = (int)(i - (long long)g * fp);
      if (c < f) v = __bfloat162float(b1[(long long)g * f + c]);
    } else {
      const long long j = i - n1;
      const int g = (int)(j / dp), c = (int)(j - (long long)g * dp);
      if (c < d) v = __bfloat162float(b2[(long long)g * d + c]);
    }
    out[i] = v;
  }
}

}  // namespace

bool tc_available() { return encode_fn() != nullptr; }

// Upper bound on ROWS pair-tiles: every expert may add one half-used pair.
static long long rows_pairs_upper(int64_t R_cap, int El) { return R_cap / 256 + El; }

// ---------------------------------------------------------------- dense helper (gate backward)
// out [rows, N] bf16 = A [rows, K] . B [N, K]^T, both K-major bf16, one row segment
// (offsets_dev = {0, rows_pad}, rows_pad = rows rounded up to 128).  Used for dL W_g^T.
cudaError_t tc_dense_store(const moe_ctx* c, const void* A, long long rows, int K, const void* B, int N, void* out,
                           const int* offsets_dev, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const long long rows_pad = (rows + BM - 1) / BM * BM;
  CUtensorMap mA, mB, mO;
  if (!make_map(&mA, A, rows, K, K, 64, BM) || !make_map(&mB, B, N, K, K, 64, BNH) ||
      !make_store_map(&mO, out, rows, N))
    return cudaErrorInvalidValue;
  TcParams p{};
  p.G = 1; p.offsets = offsets_dev; p.rows_cap = (int)rows_pad;
  p.N = N; p.K = K; p.b_group_rows = 0;
  p.o1 = reinterpret_cast<bf16*>(out); p.ldo_b = N;
  return launch_tc<TEPI_STORE, false, false, false>(mA, mB, mO, mO, mO, p,
                                                    (rows_pad / 256 + 1) * ((N + BN - 1) / BN), c->sm_count, s);
}

// ---------------------------------------------------------------- step 5 / B5 on tensor cores
cudaError_t tc_expert_ffn(const moe_ctx* c, const void* x_perm, const int32_t* offsets, int64_t R_cap,
                          const void* W1, const void* b1, const void* W2, const void* b2, void* gp, void* h,
                          void* e_out, cudaStream_t s, const int32_t* arrive, const int32_t* arrive_target) {
  const int d = c->d, f = c->f, El = c->E_local;
  if (R_cap == 0) return cudaSuccess;
  const int fp = (f + 255) / 256 * 256, dp = (d + 255) / 256 * 256;
  {
    const long long n = (long long)El * (fp + (W2 ? dp : 0));
    const int blocks = (int)((n + 255) / 256 < 4 * c->sm_count ? (n + 255) / 256 : 4 * c->sm_count);
    bias_f32_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const bf16*>(b1), W2 ? reinterpret_cast<const bf16*>(b2) : nullptr,
                                           El, f, d, fp, dp, c->biasf), count_launch();
    cudaError_t e0 = cudaGetLastError();
    if (e0 != cudaSuccess) return e0;
  }
  CUtensorMap mA, mB, mO1, mO2;
  TcParams p{};
  p.G = El; p.offsets = offsets; p.rows_cap = (int)R_cap;
  p.arrive = arrive; p.arrive_target = arrive_target; p.flags = c->flags;   // GEMM1 only (reads x_perm)
  // GEMM1: a = x_perm W1^T + b1, h = GELU(a)      A [R, d] K-major, B = W1 [El*f, d] K-major
  if (!make_map(&mA, x_perm, R_cap, d, d, 64, BM) || !make_map(&mB, W1, (long long)El * f, d, d, 64, BNH) ||
      (gp && !make_store_map(&mO1, gp, R_cap, f)) || !make_store_map(&mO2, h, R_cap, f))
    return cudaErrorInvalidValue;
  p.N = f; p.K = d; p.b_group_rows = f;
  p.bias = c->biasf; p.bias_g = fp;
  p.o1 = reinterpret_cast<bf16*>(gp ? gp : h); p.o2 = reinterpret_cast<bf16*>(h); p.ldo_b = f;
  // h above gp in memory (the layer allocates them as one [2][R_cap][f] buffer): one 3D store of
  // both staged boxes per chunk instead of two 2D stores
  p.o12 = gp && !getenv("MOE_NO_STORE_PAIR") && reinterpret_cast<uintptr_t>(h) > reinterpret_cast<uintptr_t>(gp) &&
          make_store_map_pair(&mO1, gp, R_cap, f,
                              (long long)(reinterpret_cast<uintptr_t>(h) - reinterpret_cast<uintptr_t>(gp)));
  const long long up = rows_pairs_upper(R_cap, El);
  // 4 GELU epilogue warps per lane quarter below d = 1024 (the short mainloop leaves the epilogue
  // exposed: C5 step 0 -4.6% cycles, C2 -1.4%), 3 from d = 1024 up (C4: +2.9% with 4);
  // profiles/r02/ab_gelu_epq.txt
  const long long jobs = up * ((f + BN - 1) / BN);
  cudaError_t e;
  if (d < 1024)
    e = gp ? launch_tc<TEPI_BIAS_GELU, false, false, false, 4>(mA, mB, mO1, mO2, mO1, p, jobs, c->sm_count, s)
           : launch_tc<TEPI_BIAS_GELU_H, false, false, false, 4>(mA, mB, mO2, mO2, mO2, p, jobs, c->sm_count, s);
  else
    e = gp ? launch_tc<TEPI_BIAS_GELU, false, false, false>(mA, mB, mO1, mO2, mO1, p, jobs, c->sm_count, s)
           : launch_tc<TEPI_BIAS_GELU_H, false, false, false>(mA, mB, mO2, mO2, mO2, p, jobs, c->sm_count, s);
  if (e != cudaSuccess) return e;
  if (!W2) return cudaSuccess;          // recompute call: GEMM1 only
  p.arrive = nullptr;
  // GEMM2: e_out = h W2^T + b2                     A [R, f] K-major, B = W2 [El*d, f] K-major
  if (!make_map(&mA, h, R_cap, f, f, 64, BM) || !make_map(&mB, W2, (long long)El * d, f, f, 64, BNH) ||
      !make_store_map(&mO1, e_out, R_cap, d))
    return cudaErrorInvalidValue;
  p.N = d; p.K = f; p.b_group_rows = d;
  p.bias = c->biasf + (long long)El * fp; p.bias_g = dp;
  p.o1 = reinterpret_cast<bf16*>(e_out); p.o2 = nullptr; p.ldo_b = d;
  return launch_tc<TEPI_BIAS, false, false, false>(mA, mB, mO1, mO1, mO1, p, up * ((d + BN - 1) / BN),
                                                   c->sm_count, s);
}

cudaError_t tc_expert_ffn_bwd(const moe_ctx* c, const void* d_eout, const void* x_perm, const void* gp,
                              const void* h, const int32_t* offsets, int64_t R_cap, const void* W1,
                              const void* W2, void* da, void* dx_perm, float* dW1, float* dW2, float* db1,
                              cudaStream_t s) {
  const int d = c->d, f = c->f, El = c->E_local;
  CUtensorMap mA, mB, mO, mX;
  cudaError_t e;
  if (R_cap == 0) {   // no rows at all: every expert gradient is zero
    if ((e = cudaMemsetAsync(db1, 0, sizeof(float) * El * f, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(dW1, 0, sizeof(float) * El * f * d, s)) != cudaSuccess) return e;
    return cudaMemsetAsync(dW2, 0, sizeof(float) * El * d * f, s);
  }
  const long long up = rows_pairs_upper(R_cap, El);
  {
    TcParams p{};
    p.G = El; p.offsets = offsets; p.rows_cap = (int)R_cap;
    // dgrad2: da = (d_eout W2_e) (.) GELU'(a)   A = d_eout [R, d] K-major; B(k=d, n=f) = W2 [El*d, f] MN-major
    if (!make_map(&mA, d_eout, R_cap, d, d, 64, BM) || !make_map_mn(&mB, W2, (long long)El * d, f, f, p.b3d) ||
        !make_store_map(&mO, da, R_cap, f) || !make_store_map(&mX, gp, R_cap, f))
      return cudaErrorInvalidValue;
    p.N = f; p.K = d; p.b_group_rows = d;
    p.o1 = reinterpret_cast<bf16*>(da); p.ldo_b = f;
    // db1 partials live in dx_perm's memory until dgrad1 overwrites it ([R_cap/32][f] fp32 <= R_cap x d bf16)
    const bool fuse_db1 = db1 && (long long)f * 4 <= (long long)d * 2 * 32;
    p.colpart = fuse_db1 ? reinterpret_cast<float*>(dx_perm) : nullptr;
    // 2 epilogue warps per lane quarter from d = 768 up (smaller staging -> 5 operand stages instead
    // of 4: dgrad2 -6% cycles at C2 / C3, -9% at C4), 3 below (C5's d = 512: +17% with 2;
    // profiles/r01/s2/ab_epilogue_components.txt)
    e = d >= 768 ? launch_tc<TEPI_GELU_BWD, false, true, false, 2>(mA, mB, mO, mO, mX, p, up * ((f + BN - 1) / BN),
                                                                   c->sm_count, s)
                 : launch_tc<TEPI_GELU_BWD, false, true, false>(mA, mB, mO, mO, mX, p, up * ((f + BN - 1) / BN),
                                                                c->sm_count, s);
    if (e != cudaSuccess) return e;
    if (fuse_db1) {
      if ((e = launch_db1_reduce(reinterpret_cast<const float*>(dx_perm), f, offsets, El, db1, c->colpart, R_cap, s)) !=
          cudaSuccess)
        return e;
    } else if (db1) {
      if ((e = launch_colsum_grouped(da, 1, f, offsets, El, db1, c->colpart, s)) != cudaSuccess) return e;
    }
    p.colpart = nullptr;
    // dgrad1: dx_perm = da W1_e                 A = da [R, f] K-major; B(k=f, n=d) = W1 [El*f, d] MN-major
    if (!make_map(&mA, da, R_cap, f, f, 64, BM) || !make_map_mn(&mB, W1, (long long)El * f, d, d, p.b3d) ||
        !make_store_map(&mO, dx_perm, R_cap, d))
      return cudaErrorInvalidValue;
    p.N = d; p.K = f; p.b_group_rows = f;
    p.o1 = reinterpret_cast<bf16*>(dx_perm); p.ldo_b = d;
    e = launch_tc<TEPI_STORE, false, true, false>(mA, mB, mO, mO, mO, p, up * ((d + BN - 1) / BN), c->sm_count, s);
    if (e != cudaSuccess) return e;
  }
  // wgrad2: dW2_e [d, f] = d_eout_e^T h_e       A(m=d, k=row) = d_eout MN-major; B(k=row, n=f) = h MN-major
  TcParams q{};
  q.G = El; q.offsets = offsets; q.rows_cap = (int)R_cap;
  if (!make_map_mn(&mA, d_eout, R_cap, d, d, q.a3d) || !make_map_mn(&mB, h, R_cap, f, f, q.b3d))
    return cudaErrorInvalidValue;
  q.M = d; q.N = f; q.out = dW2; q.ldo = f; q.out_g = (long long)d * f;
  if (!make_store_map_f32(&mO, dW2, (long long)El * d, f)) return cudaErrorInvalidValue;
  e = launch_tc<TEPI_F32, true, true, true>(mA, mB, mO, mO, mO, q,
                                            (long long)El * ((d + 255) / 256) * ((f + BN - 1) / BN), c->sm_count, s);
  if (e != cudaSuccess) return e;
  // wgrad1: dW1_e [f, d] = da_e^T x_perm_e      A(m=f, k=row) = da MN-major; B(k=row, n=d) = x_perm MN-major
  if (!make_map_mn(&mA, da, R_cap, f, f, q.a3d) || !make_map_mn(&mB, x_perm, R_cap, d, d, q.b3d))
    return cudaErrorInvalidValue;
  q.M = f; q.N = d; q.out = dW1; q.ldo = d; q.out_g = (long long)f * d;
  if (!make_store_map_f32(&mO, dW1, (long long)El * f, d)) return cudaErrorInvalidValue;
  return launch_tc<TEPI_F32, true, true, true>(mA, mB, mO, mO, mO, q,
                                               (long long)El * ((f + 255) / 256) * ((d + BN - 1) / BN), c->sm_count,
                                               s);
}

}  // namespace moe
