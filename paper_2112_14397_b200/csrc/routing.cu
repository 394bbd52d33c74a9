// routing.cu -- step 4 (dispatch: scan + stable permute), step 6 (combine), their
// backward passes (combine_bwd, dispatch_bwd) and step 6b (expert-diversify spawn).
// All HBM-bound: 16-byte vector loads/stores, fp32 accumulation, fixed summation order.
#include "common.cuh"
#include "internal.h"

namespace moe {

namespace {

// ------------------------------------------------------------------ scan
// One CTA per expert over the expert-major per-block counts blk_cnt[E][nblk]: thread i takes
// block b0 + i of each blockDim-block chunk (coalesced; blockDim = nblk rounded up to a warp, <= 1024), a block scan (warp scans + the warp totals
// in shared memory) gives the exclusive per-block bases blk_base[E][nblk], chained across chunks
// by a carry; the expert total goes to tot[e].  The last CTA to finish (ticket counter in the
// flags word kScanTicket, reset by that CTA) forms the 128-aligned exclusive prefix of the
// totals -> offsets[E+1].  Integer arithmetic only (deterministic).
constexpr int kScanThreads = 1024;
constexpr int kScanTicket = 12;
static inline int scan_threads(int nblk) { return nblk >= kScanThreads ? kScanThreads : (nblk < 32 ? 32 : (nblk + 31) / 32 * 32); }
__global__ void __launch_bounds__(kScanThreads) dispatch_scan_kernel(const int* __restrict__ blk_cnt, int nblk, int E,
                                                                     int* __restrict__ blk_base, int* __restrict__ tot,
                                                                     int* __restrict__ offsets, int* __restrict__ R_out,
                                                                     long long R_cap, int* __restrict__ flags) {
  __shared__ int s_w[32];
  __shared__ bool s_last;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int e = blockIdx.x;
  const int* src = blk_cnt + (long long)e * nblk;
  int* dst = blk_base + (long long)e * nblk;
  int carry = 0;
  const int nw = blockDim.x / 32;
  for (int b0 = 0; b0 < nblk; b0 += (int)blockDim.x) {
    const int b = b0 + (int)threadIdx.x;
    const int v = b < nblk ? src[b] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += n;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      int w = lane < nw ? s_w[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += n;
      }
      s_w[lane] = w;                                   // inclusive prefix of the warp totals
    }
    __syncthreads();
    const int wbase = warp ? s_w[warp - 1] : 0;
    if (b < nblk) dst[b] = carry + wbase + inc - v;
    carry += s_w[nw - 1];
    __syncthreads();                                   // s_w is rewritten by the next chunk
  }
  if (threadIdx.x == 0) {
    tot[e] = carry;
    __threadfence();
    s_last = atomicAdd(&flags[kScanTicket], 1) == E - 1;
  }
  __syncthreads();
  if (s_last && warp == 0) {
    // the totals of all E (<= 128) experts, loaded together (4 per lane, L2-coherent loads),
    // aligned to 128 rows and scanned by one warp
    __threadfence();
    int a[4], asum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int g = 4 * lane + q;
      a[q] = g < E ? (__ldcg(tot + g) + kRowAlign - 1) / kRowAlign * kRowAlign : 0;
      asum += a[q];
    }
    int inc = asum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += n;
    }
    int run = inc - asum;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int g = 4 * lane + q;
      if (g < E) offsets[g] = run;
      run += a[q];
    }
    const int R = __shfl_sync(0xffffffffu, inc, 31);
    if (lane == 0) {
      flags[kScanTicket] = 0;                          // ready for the next launch on this stream
      offsets[E] = R;
      *R_out = R;
      if ((long long)R > R_cap) {
        atomicOr(&flags[0], kFlagCapacity);
        flags[2] = R;
      }
    }
  }
}

// Small inputs (nblk <= kScanSmallBlocks: C2/C3/C5) take one CTA of 1024 threads, warp per
// expert, each lane 4 consecutive blocks per 128-block step (coalesced), warp scan of lane
// totals, then thread 0 forms the offsets: one launch phase, ~2 us, where the per-expert
// CTAs above pay a second (ticket + L2 round trip) phase.
constexpr int kScanSmallBlocks = 256;
__global__ void __launch_bounds__(1024) dispatch_scan_small_kernel(const int* __restrict__ blk_cnt, int nblk, int E,
                                                            int* __restrict__ blk_base, int* __restrict__ tot,
                                                            int* __restrict__ offsets, int* __restrict__ R_out,
                                                            long long R_cap, int* __restrict__ flags) {
  __shared__ int s_tot[128];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int e = warp; e < E; e += nw) {
    const int* src = blk_cnt + (long long)e * nblk;
    int* dst = blk_base + (long long)e * nblk;
    int carry = 0;
    for (int b0 = 0; b0 < nblk; b0 += 128) {
      const int b = b0 + lane * 4;
      int v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (b + q < nblk) ? src[b + q] : 0;
      const int lsum = v[0] + v[1] + v[2] + v[3];
      int inc = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
      }
      int run = carry + inc - lsum;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (b + q < nblk) dst[b + q] = run;
        run += v[q];
      }
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) s_tot[e] = carry;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long off = 0;
    for (int e = 0; e < E; ++e) {
      offsets[e] = (int)off;
      tot[e] = s_tot[e];
      off += (long long)(s_tot[e] + kRowAlign - 1) / kRowAlign * kRowAlign;
    }
    offsets[E] = (int)off;
    *R_out = (int)off;
    if (off > R_cap) {
      atomicOr(&flags[0], kFlagCapacity);
      flags[2] = (int)off;
    }
  }
}

// per-block bases + 128-aligned expert offsets from the gate's per-block counts
static void launch_dispatch_scan(const moe_ctx* c, int* offsets, int* R_out, long long R_cap, cudaStream_t s) {
  if (c->nblk <= kScanSmallBlocks)
    dispatch_scan_small_kernel<<<1, 1024, 0, s>>>(c->blk_cnt, c->nblk, c->E, c->blk_base, c->tot, offsets, R_out, R_cap,
                                                  c->flags), count_launch();
  else
    dispatch_scan_kernel<<<c->E, scan_threads(c->nblk), 0, s>>>(c->blk_cnt, c->nblk, c->E, c->blk_base, c->tot,
                                                                 offsets, R_out, R_cap, c->flags), count_launch();
}

// ------------------------------------------------------------------ permute
// Rank pass: one CTA per gate block of kGateBT tokens.  Each warp ballots every expert over
// its 32 tokens (no block barrier per expert); one barrier; then a token's row for expert e is
//   offsets[e] + blk_base[e][blk] + (selected tokens of e in lower warps) + (lower lanes).
// The first two terms are staged in shared memory while the flags load; each thread keeps a
// bitmask of its selected experts and walks only those, 8 at a time with their probs loads
// issued together (the pass is latency-bound: 1-2 memory round trips per token, not one per
// selected expert).  Writes slot (row index), row_token, row_gate; zeroes the pad rows of
// expert blockIdx.x, ...
template <typename T>
__global__ void __launch_bounds__(kGateBT) dispatch_rank_kernel(
    const float* __restrict__ probs, int* __restrict__ slot, int T_, int d, int E, const int* __restrict__ blk_base,
    const int* __restrict__ offsets, const int* __restrict__ tot, T* __restrict__ x_perm, int* __restrict__ row_token,
    float* __restrict__ row_gate, long long R_cap) {
  __shared__ unsigned s_bal[kGateBT / 32][128];
  __shared__ int s_base[128];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int t = blockIdx.x * kGateBT + tid;
  const bool valid = t < T_;
  for (int e = tid; e < E; e += kGateBT) s_base[e] = offsets[e] + blk_base[(long long)e * gridDim.x + blockIdx.x];
  // 16 selection flags per thread in flight (16-byte loads when the rows allow), then 16 ballots
  const bool vec = (E & 3) == 0;
  unsigned selm[4] = {0u, 0u, 0u, 0u};              // this thread's selected experts (E <= 128)
  for (int e0 = 0; e0 < E; e0 += 16) {
    int v[16];
    if (vec && e0 + 16 <= E) {
      int4 q[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        q[i] = make_int4(-1, -1, -1, -1);
        if (valid) q[i] = *reinterpret_cast<const int4*>(slot + (long long)t * E + e0 + 4 * i);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) { v[4 * i] = q[i].x; v[4 * i + 1] = q[i].y; v[4 * i + 2] = q[i].z; v[4 * i + 3] = q[i].w; }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = (valid && e0 + j < E) ? slot[(long long)t * E + e0 + j] : -1;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const bool sel = v[j] >= 0 && e0 + j < E;
      const unsigned bal = __ballot_sync(0xffffffffu, sel);
      if (lane == 0 && e0 + j < E) s_bal[warp][e0 + j] = bal;
      if (sel) selm[(e0 + j) >> 5] |= 1u << ((e0 + j) & 31);
    }
  }
  __syncthreads();
  if (valid) {
    const unsigned lower = (1u << lane) - 1u;
    int word = 0;
    unsigned bits = selm[0];
    while (true) {
      // next batch of up to 8 selected experts
      int es[8], nb = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        while (bits == 0u && word < 3) bits = selm[++word];
        es[j] = -1;
        if (bits) {
          es[j] = word * 32 + __ffs(bits) - 1;
          bits &= bits - 1u;
          ++nb;
        }
      }
      if (nb == 0) break;
      float pg[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) pg[j] = es[j] >= 0 ? probs[(long long)t * E + es[j]] : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = es[j];
        if (e < 0) continue;
        const unsigned mine = s_bal[warp][e];
        int wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += __popc(s_bal[w][e]);
        const int row = s_base[e] + wpre + __popc(mine & lower);
        if (row < R_cap) {
          slot[(long long)t * E + e] = row;
          row_token[row] = t;
          row_gate[row] = pg[j];
        } else {
          slot[(long long)t * E + e] = -1;   // dropped (MOE_ECAPACITY raised by the scan)
        }
      }
      if (nb < 8) break;
    }
  }
  // pad rows of experts e = blockIdx.x, blockIdx.x + gridDim.x, ...: zero
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const long long r0 = (long long)offsets[e] + tot[e], r1 = offsets[e + 1];
    for (long long r = r0 + warp; r < r1 && r < R_cap; r += kGateBT / 32) {
      if (lane == 0) { row_token[r] = -1; row_gate[r] = 0.f; }
      T* dst = x_perm + r * d;
      for (int v = lane; v < nvec; v += 32) st_v4(dst + (long long)v * V, make_uint4(0, 0, 0, 0));
    }
  }
}

// Copy pass: one warp per token; x_t is read once (4 x 16 B per lane in flight) and stored
// to each of its selected rows (found with ballots over the final slot row).
template <typename T>
__global__ void __launch_bounds__(256) dispatch_copy_kernel(const T* __restrict__ x, const int* __restrict__ slot,
                                                            int T_, int d, int E, T* __restrict__ x_perm) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t = blockIdx.x * 8 + warp;
  if (t >= T_) return;
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  const T* src = x + (long long)t * d;
  const int* srow = slot + (long long)t * E;
  for (int v0 = 0; v0 < nvec; v0 += 32 * 4) {
    uint4 buf[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int v = v0 + q * 32 + lane;
      if (v < nvec) buf[q] = ld_nc_v4(src + (long long)v * V);
    }
    for (int g = 0; g < E; g += 32) {
      const int sv = (g + lane < E) ? srow[g + lane] : -1;
      unsigned bal = __ballot_sync(0xffffffffu, sv >= 0);
      while (bal) {
        const int b = __ffs(bal) - 1;
        bal &= bal - 1;
        const int row = __shfl_sync(0xffffffffu, sv, b);
        T* dst = x_perm + (long long)row * d;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int v = v0 + q * 32 + lane;
          if (v < nvec) st_v4(dst + (long long)v * V, buf[q]);
        }
      }
    }
  }
}

// ------------------------------------------------------------------ combine
// One warp per token.  The token's selected rows are found with ballots over its slot row
// (ascending expert order is the bit order), so the work is O(selected), not O(E).
// Columns are processed 4 x 16-byte vectors per lane at a time (independent loads in flight).
// Row sources of the gather: this device's row layout (row r of `rows`, weight row_gate[r]),
// or the expert-parallel peer layouts (row r of the layout on the rank owning expert e, reached
// through NVLink peer pointers; weight = the token's probs[e]).
template <typename T>
struct LocalRows {
  const T* rows;
  const float* gate;
  int d;
  __device__ __forceinline__ const T* row(int, int r) const { return rows + (long long)r * d; }
  __device__ __forceinline__ float weight(int, int r) const { return gate[r]; }
};
template <typename T>
struct PeerRows {
  const PeerTable* peers;      // [rank] -> row layout base on that rank
  const float* probs_t;        // this token's probs row (weights of its selected experts)
  int d, El;
  __device__ __forceinline__ const T* row(int e, int r) const {
    return reinterpret_cast<const T*>(peers->p[e / El]) + (long long)r * d;
  }
  __device__ __forceinline__ float weight(int e, int) const { return probs_t[e]; }
};

// the whole slot row of a token (E <= 128: up to 4 entries per lane), one memory round trip
__device__ __forceinline__ void load_slot_row(const int* __restrict__ slot_row, int E, int lane, int (&svs)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) svs[i] = (32 * i < E && 32 * i + lane < E) ? slot_row[32 * i + lane] : -1;
}

template <typename T, bool WEIGHTED, typename TX = float, int QV = 4, typename Src = LocalRows<T>>
__device__ __forceinline__ void gather_sum_token_sv(const Src& src, const int (&svs)[4], int d, int E,
                                                    const TX* extra, T* out, int lane) {
  // `extra` may alias `out` (the accumulating dispatch backward): each lane loads its own
  // elements of the row with coherent loads before it stores them
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  constexpr bool TWO = QV <= 3;                     // two rows in flight when registers allow
  for (int v0 = 0; v0 < nvec; v0 += 32 * QV) {
    float acc[QV][V];
#pragma unroll
    for (int q = 0; q < QV; ++q)
#pragma unroll
      for (int k = 0; k < V; ++k) acc[q][k] = 0.f;
    if (extra) {                                      // the extra row term starts the sum (loads issued first)
#pragma unroll
      for (int q = 0; q < QV; ++q) {
        const int v = v0 + q * 32 + lane;
        if (v < nvec) {
          if (sizeof(TX) == 2) {
            unpack16(ld_v4(extra + (long long)v * V), acc[q], bf16());
          } else {
#pragma unroll
            for (int h = 0; h < V / 4; ++h)
              unpack16(ld_v4(reinterpret_cast<const float*>(extra) + (long long)v * V + 4 * h), acc[q] + 4 * h, float());
          }
        }
      }
    }
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
      const int g = 32 * gi;
      if (g >= E) break;                               // warp-uniform
      const int sv = svs[gi];
      unsigned bal = __ballot_sync(0xffffffffu, sv >= 0);
      while (bal) {
        // two selected rows per pass (both rows' loads in flight), accumulated in ascending e
        const int b = __ffs(bal) - 1;
        bal &= bal - 1;
        const bool two = TWO && bal != 0;
        const int b2 = two ? __ffs(bal) - 1 : b;
        if (two) bal &= bal - 1;
        const int r = __shfl_sync(0xffffffffu, sv, b);
        const int r2 = __shfl_sync(0xffffffffu, sv, b2);
        const float gw = WEIGHTED ? src.weight(g + b, r) : 1.0f;
        const float gw2 = WEIGHTED && two ? src.weight(g + b2, r2) : 1.0f;
        const T* p1 = src.row(g + b, r);
        const T* p2 = src.row(g + b2, r2);
        uint4 raw[QV], raw2[QV];
#pragma unroll
        for (int q = 0; q < QV; ++q) {
          const int v = v0 + q * 32 + lane;
          if (v < nvec) {
            raw[q] = ld_nc_v4(p1 + (long long)v * V);
            if (two) raw2[q] = ld_nc_v4(p2 + (long long)v * V);
          }
        }
#pragma unroll
        for (int q = 0; q < QV; ++q) {
          const int v = v0 + q * 32 + lane;
          if (v < nvec) {
            float o[V];
            unpack16(raw[q], o, T());
#pragma unroll
            for (int k = 0; k < V; ++k) acc[q][k] = WEIGHTED ? fmaf(gw, o[k], acc[q][k]) : acc[q][k] + o[k];
            if (two) {
              unpack16(raw2[q], o, T());
#pragma unroll
              for (int k = 0; k < V; ++k) acc[q][k] = WEIGHTED ? fmaf(gw2, o[k], acc[q][k]) : acc[q][k] + o[k];
            }
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < QV; ++q) {
      const int v = v0 + q * 32 + lane;
      if (v < nvec) {
        st_v4(out + (long long)v * V, pack16(acc[q], T()));
      }
    }
  }
}

template <typename T, bool WEIGHTED, typename TX = float, int QV = 4, typename Src = LocalRows<T>>
__device__ __forceinline__ void gather_sum_token(const Src& src, const int* __restrict__ slot_row, int d, int E,
                                                 const TX* extra, T* out, int lane) {
  int svs[4];
  load_slot_row(slot_row, E, lane, svs);
  gather_sum_token_sv<T, WEIGHTED, TX, QV, Src>(src, svs, d, E, extra, out, lane);
}

// y[t] = sum_{e asc} row_gate[r] * e_out[r], r = slot[t,e].  A warp takes two consecutive
// tokens and loads both slot rows up front, so the second token's slot round trip hides under
// the first token's row loads (the dispatch backward hides it under its dx-row loads): C4
// 109 -> 98 us, C5 step 19 8.5 -> 7.7 us.  Not at QV = 3 (d = 768: the extra registers spill,
// C2 +6%).
template <int QV> constexpr int combine_tpw() { return QV == 3 ? 1 : 2; }
template <typename T, int QV>
__global__ void __launch_bounds__(256, 4) combine_kernel(const T* __restrict__ e_out, const float* __restrict__ row_gate,
                                                      const int* __restrict__ slot, int T_, int d, int E,
                                                      T* __restrict__ y) {
  constexpr int TPW = combine_tpw<QV>();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t0 = (blockIdx.x * 8 + warp) * TPW;
  if (t0 >= T_) return;
  int sv[TPW][4];
#pragma unroll
  for (int j = 0; j < TPW; ++j)
    if (t0 + j < T_) load_slot_row(slot + (long long)(t0 + j) * E, E, lane, sv[j]);
#pragma unroll
  for (int j = 0; j < TPW; ++j)
    if (t0 + j < T_)
      gather_sum_token_sv<T, true, float, QV>(LocalRows<T>{e_out, row_gate, d}, sv[j], d, E, (const float*)nullptr,
                                              y + (long long)(t0 + j) * d, lane);
}
// vectors per lane per pass: the whole row in one pass up to 4 x 16 B per lane
static inline int pass_vectors(int d, int V) {
  const int q = (d / V + 31) / 32;
  return q < 1 ? 1 : (q > 4 ? 4 : q);
}

// ------------------------------------------------------------------ combine backward
// One warp per row r < offsets[E]: d_eout[r] = g dy[t]; dG_row[r] = <dy[t], e_out[r]>.
template <typename T, bool PEER = false>
__global__ void __launch_bounds__(256) combine_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ e_out,
                                                          const float* __restrict__ row_gate,
                                                          const int* __restrict__ row_token,
                                                          const int* __restrict__ offsets, int E, int d,
                                                          long long R_cap, T* __restrict__ d_eout,
                                                          float* __restrict__ dG_row,
                                                          const int* __restrict__ row_src,
                                                          const __grid_constant__ PeerTable dyp) {
  // PEER (peer-memory EP, rows wider than the fused kernel's registers): the row's token lives
  // on rank row_src[r] and its dy row is read through that rank's peer pointer
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long r = (long long)blockIdx.x * 8 + warp;
  const long long R = min((long long)offsets[E], R_cap);
  if (r >= R) return;
  const int t = row_token[r];
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  T* dst = d_eout + r * d;
  if (t < 0) {
    for (int v = lane; v < nvec; v += 32) st_v4(dst + (long long)v * V, make_uint4(0, 0, 0, 0));
    if (lane == 0) dG_row[r] = 0.f;
    return;
  }
  const T* dyt = (PEER ? reinterpret_cast<const T*>(dyp.p[row_src[r]]) : dy) + (long long)t * d;
  const float gw = row_gate[r];
  float dot = 0.f;
  for (int v = lane; v < nvec; v += 32) {
    float a[V], b[V], o[V];
    unpack16(ld_nc_v4(dyt + (long long)v * V), a, T());
    unpack16(ld_nc_v4(e_out + r * d + (long long)v * V), b, T());
#pragma unroll
    for (int k = 0; k < V; ++k) {
      dot = fmaf(a[k], b[k], dot);
      o[k] = gw * a[k];
    }
    st_v4(dst + (long long)v * V, pack16(o, T()));
  }
  dot = warp_sum(dot);
  if (lane == 0) dG_row[r] = dot;
}

// Fused variant (single rank, d <= 32 * MAXV * V): block (s, g) owns split s of expert g's
// rows [offsets[g], offsets[g+1]) (8 warps, warp w takes rows r0 + w, r0 + w + 8, ...), writes
// d_eout / dG_row exactly as above and also the db2 column-sum partial of its rows,
// part[g][s][n] = sum of the stored (rounded) d_eout[r][n], warps combined in fixed order.
// The dy and e_out rows stream through a per-warp ring of CB_NB shared-memory stages filled
// by cp.async (16 B per lane and vector, each lane reads back only its own vectors, so no
// cross-lane synchronisation): CB_NB - 1 rows per warp are in flight while one is computed,
// without holding them in registers.  Each lane's column sums (its MAXV * V columns) stay in
// registers; row metadata is loaded one row ahead of its copies.
// COMPUTE = false: only the partials, from an existing d_eout (same row partition and summation
// order, so both paths give bit-identical db2).
// PEER (fused peer-memory EP, expert side): the row's token lives on rank row_src[r]; its dy
// row is read through that rank's NVLink peer pointer dyp.p[row_src[r]] (no dy exchange).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// ring depth per MAXV: ~96 KB of stages per 256-thread block (2 blocks / SM)
template <int MAXV> struct CbDepth { static constexpr int N = MAXV == 1 ? 8 : (MAXV == 2 ? 6 : (MAXV == 3 ? 4 : 3)); };
template <int MAXV> constexpr size_t cb_smem_bytes() {
  return (size_t)8 * CbDepth<MAXV>::N * 2 * MAXV * 32 * 16 + 8 * CbDepth<MAXV>::N * sizeof(int2);
}

template <typename T, int MAXV, bool COMPUTE, bool PEER = false>
__global__ void __launch_bounds__(256, 2) combine_bwd_colsum_kernel(const T* __restrict__ dy, const T* __restrict__ e_out,
                                                                 const float* __restrict__ row_gate,
                                                                 const int* __restrict__ row_token,
                                                                 const int* __restrict__ offsets, int d,
                                                                 long long R_cap, int S, T* __restrict__ d_eout,
                                                                 float* __restrict__ dG_row, float* __restrict__ part,
                                                                 const int* __restrict__ row_src,
                                                                 const __grid_constant__ PeerTable dyp) {
  constexpr int V = Vec16<T>::N;
  constexpr int NB = CbDepth<MAXV>::N;
  constexpr int STAGE = 2 * MAXV * 32;              // uint4 per warp stage: [dy | e_out][MAXV][32 lanes]
  extern __shared__ uint4 cb_smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int s = blockIdx.x, g = blockIdx.y;
  const long long off0 = offsets[g], off1 = min((long long)offsets[g + 1], R_cap);
  const long long len = off1 > off0 ? off1 - off0 : 0;
  const long long per = ((len + S - 1) / S + 7) / 8 * 8;
  const long long r0 = off0 + (long long)s * per, r1 = min(off1, r0 + per);
  const int nvec = d / V;
  const long long nrows = r1 > r0 + warp ? (r1 - r0 - warp + 7) / 8 : 0;   // rows r0 + warp + 8k
  uint4* ring = cb_smem + (size_t)warp * NB * STAGE;
  int2* meta = reinterpret_cast<int2*>(cb_smem + (size_t)8 * NB * STAGE) + warp * NB;   // (token, gate bits)
  float acc[MAXV * V];
#pragma unroll
  for (int i = 0; i < MAXV * V; ++i) acc[i] = 0.f;

  if (!COMPUTE) {
    for (long long k = 0; k < nrows; ++k) {
      const T* src = d_eout + (r0 + warp + 8 * k) * d;
#pragma unroll
      for (int j = 0; j < MAXV; ++j) {
        const int v = lane + 32 * j;
        if (v < nvec) {
          float o[V];
          unpack16(ld_nc_v4(src + (long long)v * V), o, T());
#pragma unroll
          for (int h = 0; h < V; ++h) acc[j * V + h] += o[h];
        }
      }
    }
  } else {
    // metadata of the next row to issue (one row ahead of its copies)
    int t_nx = -1, q_nx = 0;
    float g_nx = 0.f;
    if (nrows > 0) {
      t_nx = row_token[r0 + warp];
      g_nx = row_gate[r0 + warp];
      if (PEER) q_nx = row_src[r0 + warp];
    }
    auto issue = [&](long long k) {
      if (k < nrows) {
        const long long r = r0 + warp + 8 * k;
        const int b = (int)(k % NB);
        const int t = t_nx;
        meta[b] = make_int2(t, __float_as_int(g_nx));   // every lane stores the same value
        if (t >= 0) {
          const T* dyb = PEER ? reinterpret_cast<const T*>(dyp.p[q_nx]) : dy;
          uint4* st = ring + b * STAGE;
#pragma unroll
          for (int j = 0; j < MAXV; ++j) {
            const int v = lane + 32 * j;
            if (v < nvec) {
              cp_async16(st + j * 32 + lane, dyb + (long long)t * d + (long long)v * V);
              cp_async16(st + (MAXV + j) * 32 + lane, e_out + r * d + (long long)v * V);
            }
          }
        }
        if (k + 1 < nrows) {
          t_nx = row_token[r + 8];
          g_nx = row_gate[r + 8];
          if (PEER) q_nx = row_src[r + 8];
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int k = 0; k < NB - 1; ++k) issue(k);
    for (long long k = 0; k < nrows; ++k) {
      __syncwarp();                                 // every lane is done with row k - 1's meta slot
      issue(k + NB - 1);
      cp_async_wait<NB - 1>();                      // this lane's copies of row k have landed
      const long long r = r0 + warp + 8 * k;
      const int b = (int)(k % NB);
      const int2 m = meta[b];
      T* dst = d_eout + r * d;
      if (m.x < 0) {
#pragma unroll
        for (int j = 0; j < MAXV; ++j) {
          const int v = lane + 32 * j;
          if (v < nvec) st_v4(dst + (long long)v * V, make_uint4(0, 0, 0, 0));
        }
        if (lane == 0) dG_row[r] = 0.f;
        continue;
      }
      const float gw = __int_as_float(m.y);
      const uint4* st = ring + b * STAGE;
      float dot = 0.f;
#pragma unroll
      for (int j = 0; j < MAXV; ++j) {
        const int v = lane + 32 * j;
        if (v < nvec) {
          float a[V], bb[V], o[V];
          unpack16(st[j * 32 + lane], a, T());
          unpack16(st[(MAXV + j) * 32 + lane], bb, T());
#pragma unroll
          for (int h = 0; h < V; ++h) {
            dot = fmaf(a[h], bb[h], dot);
            o[h] = gw * a[h];
          }
          const uint4 w = pack16(o, T());
          st_v4(dst + (long long)v * V, w);
          unpack16(w, o, T());                      // the stored (rounded) values
#pragma unroll
          for (int h = 0; h < V; ++h) acc[j * V + h] += o[h];
        }
      }
      dot = warp_sum(dot);
      if (lane == 0) dG_row[r] = dot;
    }
    cp_async_wait<0>();
  }
  // block partial: warp sums through shared memory (the ring is free now), added in warp order
  __syncthreads();
  float* red = reinterpret_cast<float*>(cb_smem);   // [8][d]
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    const int v = lane + 32 * j;
    if (v < nvec) {
#pragma unroll
      for (int h = 0; h < V; h += 4)
        *reinterpret_cast<float4*>(red + warp * d + v * V + h) =
            make_float4(acc[j * V + h], acc[j * V + h + 1], acc[j * V + h + 2], acc[j * V + h + 3]);
    }
  }
  __syncthreads();
  for (int n = threadIdx.x; n < d; n += 256) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w * d + n];
    part[((long long)g * S + s) * d + n] = t;
  }
}

// ------------------------------------------------------------------ dispatch backward
// One warp per token: dx[t] = dxg[t] + sum_{e asc} dx_perm[slot[t,e]]  (dxg may be NULL, or dx itself:
// the accumulating form).
template <typename T, typename TX, int QV>
__global__ void __launch_bounds__(256, 4) dispatch_bwd_kernel(const T* __restrict__ dx_perm, const int* __restrict__ slot,
                                                           const TX* dxg, int T_, int d, int E, T* dx) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t = blockIdx.x * 8 + warp;
  if (t >= T_) return;
  gather_sum_token<T, false, TX, QV>(LocalRows<T>{dx_perm, nullptr, d}, slot + (long long)t * E, d, E,
                                 dxg ? dxg + (long long)t * d : nullptr, dx + (long long)t * d, lane);
}

// ------------------------------------------------------------------ spawn (step 6b)
// Thread per 16-byte vector of W_s (V = 8 bf16 / 4 fp32 elements): the vector is read once and
// stored once per local expert with its V mask bits applied, so each warp store covers 512
// contiguous bytes of the expert's copy (a thread per 32-element mask word, the previous form,
// stored 16 B per lane at a 64 B stride: 0.43 of the HBM peak at C4).
template <typename T>
__global__ void __launch_bounds__(256) spawn_kernel(const T* __restrict__ Ws, const uint32_t* __restrict__ M,
                                                    long long n, long long words, int e0, int E_local,
                                                    T* __restrict__ W) {
  constexpr int V = Vec16<T>::N;
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long base = v * V;
  if (base >= n) return;
  if (base + V <= n) {
    const uint4 src = ld_nc_v4(Ws + base);
    const long long w = base / 32;
    const int sh = (int)(base % 32);
    for (int j = 0; j < E_local; ++j) {
      const uint32_t bits = __ldg(M + (long long)(e0 + j) * words + w) >> sh;
      uint4 o = src;
      uint32_t* po = reinterpret_cast<uint32_t*>(&o);
      if (V == 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (!((bits >> k) & 1u)) po[k] = 0u;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          po[k] &= (((bits >> (2 * k)) & 1u) ? 0x0000ffffu : 0u) | (((bits >> (2 * k + 1)) & 1u) ? 0xffff0000u : 0u);
      }
      st_v4(W + (long long)j * n + base, o);
    }
  } else {
    for (int j = 0; j < E_local; ++j)
      for (long long i = base; i < n; ++i) {
        const uint32_t bits = M[(long long)(e0 + j) * words + i / 32];
        W[(long long)j * n + i] = ((bits >> (i % 32)) & 1u) ? Ws[i] : from_f32<T>(0.f);
      }
  }
}

template <typename T>
__global__ void copy_bias_kernel(const T* __restrict__ b, int n, int E_local, T* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n * E_local) return;
  out[i] = b[i % n];
}

template <typename T>
cudaError_t spawn_typed(const moe_ctx* c, const void* W1s, const void* b1s, const void* W2s, const void* b2s,
                        const uint32_t* M1, const uint32_t* M2, void* W1, void* b1, void* W2, void* b2,
                        cudaStream_t s) {
  const long long n = (long long)c->f * c->d;
  const long long words = (n + 31) / 32;
  const int e0 = c->rank * c->E_local;
  constexpr int V = Vec16<T>::N;
  const unsigned blocks = (unsigned)(((n + V - 1) / V + 255) / 256);
  spawn_kernel<T><<<blocks, 256, 0, s>>>((const T*)W1s, M1, n, words, e0, c->E_local, (T*)W1), count_launch();
  spawn_kernel<T><<<blocks, 256, 0, s>>>((const T*)W2s, M2, n, words, e0, c->E_local, (T*)W2), count_launch();
  copy_bias_kernel<T><<<(c->f * c->E_local + 255) / 256, 256, 0, s>>>((const T*)b1s, c->f, c->E_local, (T*)b1), count_launch();
  copy_bias_kernel<T><<<(c->d * c->E_local + 255) / 256, 256, 0, s>>>((const T*)b2s, c->d, c->E_local, (T*)b2), count_launch();
  return cudaGetLastError();
}

// ================================================================== fused peer-memory EP
// Expert parallelism with the exchanges fused into the routing kernels over NVLink peer
// memory (every rank's row buffers are mapped into every other rank: symmetric memory).
// Token side writes its x rows straight into the owning rank's expert-side layout
// (ep2_copy); the combine, the gate backward and the dispatch backward gather e_out,
// dG and dx_perm rows from the owning ranks through peer loads; the expert side's
// combine_bwd reads dy rows from the token owners (combine_bwd_colsum_kernel<PEER>).
// slot[t, e] holds the row on rank e / E_local.  Layouts equal the NCCL path's.

// counts all-gather by peer stores: counts_all[me][e] on every rank
__global__ void ep2_counts_kernel(const int* __restrict__ counts, int E, int me, int W,
                                  const __grid_constant__ PeerTable all) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < W * E; i += gridDim.x * blockDim.x) {
    const int p = i / E, e = i - p * E;
    reinterpret_cast<int*>(const_cast<void*>(all.p[p]))[(long long)me * E + e] = counts[e];
  }
}

// Plan from counts_all [W][E] (identical on every rank): my recv layout (offsets [El+1],
// totals [El]) and, for my tokens, the first destination row of every global expert e:
//   base[e] = off_{e / El}[e % El] + sum_{q < me} counts_all[q][e].
__global__ void __launch_bounds__(256) ep2_plan_kernel(const int* __restrict__ counts_all, int W, int E, int me,
                                                       long long R_cap, int* __restrict__ off_me,
                                                       int* __restrict__ tot_me, int* __restrict__ base,
                                                       int* __restrict__ flags) {
  extern __shared__ long long s_tot[];             // [E] column totals
  const int El = E / W;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    long long t = 0;
    for (int q = 0; q < W; ++q) t += counts_all[(long long)q * E + e];
    s_tot[e] = t;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int p = e / El, j = e - p * El;
    long long off = 0;
    for (int j2 = 0; j2 < j; ++j2) off += (s_tot[p * El + j2] + kRowAlign - 1) / kRowAlign * kRowAlign;
    long long pre = 0;
    for (int q = 0; q < me; ++q) pre += counts_all[(long long)q * E + e];
    base[e] = (int)(off + pre);
    if (p == me) {
      off_me[j] = (int)off;
      tot_me[j] = (int)s_tot[e];
      if (j == El - 1) {
        const long long end = off + (s_tot[e] + kRowAlign - 1) / kRowAlign * kRowAlign;
        off_me[El] = (int)end;
      }
    }
    if (j == El - 1) {   // capacity of rank p's layout (every rank raises it, so each rank's check sees it)
      const long long end = off + (s_tot[e] + kRowAlign - 1) / kRowAlign * kRowAlign;
      if (end > R_cap) {
        atomicOr(&flags[0], kFlagCapacity);
        flags[2] = (int)(end < 0x7fffffff ? end : 0x7fffffff);
      }
    }
  }
}

// expert side: pad rows of my layout -> zero x, row_token -1, gate 0, source 0
template <typename T>
__global__ void ep2_prepare_kernel(T* __restrict__ x_recv, int* __restrict__ rtok, int* __restrict__ rsrc,
                                   float* __restrict__ rgate, const int* __restrict__ off, const int* __restrict__ tot,
                                   int El, int d, long long R_cap) {
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int j = blockIdx.y; j < El; j += gridDim.y) {
    const long long r0 = (long long)off[j] + tot[j], r1 = min((long long)off[j + 1], R_cap);
    for (long long r = r0 + blockIdx.x * nw + warp; r < r1; r += (long long)gridDim.x * nw) {
      if (lane == 0) { rtok[r] = -1; rsrc[r] = 0; rgate[r] = 0.f; }
      for (int v = lane; v < nvec; v += 32) st_v4(x_recv + r * d + (long long)v * V, make_uint4(0, 0, 0, 0));
    }
  }
}

// token side copy pass: x_t read once, stored into each selected expert's row on its owner
template <typename T>
__global__ void __launch_bounds__(256) ep2_copy_kernel(const T* __restrict__ x, const int* __restrict__ slot, int T_,
                                                       int d, int E, int El, const __grid_constant__ PeerTable xr) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t = blockIdx.x * 8 + warp;
  if (t >= T_) return;
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  const T* src = x + (long long)t * d;
  const int* srow = slot + (long long)t * E;
  for (int v0 = 0; v0 < nvec; v0 += 32 * 4) {
    uint4 buf[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int v = v0 + q * 32 + lane;
      if (v < nvec) buf[q] = ld_nc_v4(src + (long long)v * V);
    }
    for (int g = 0; g < E; g += 32) {
      const int sv = (g + lane < E) ? srow[g + lane] : -1;
      unsigned bal = __ballot_sync(0xffffffffu, sv >= 0);
      while (bal) {
        const int b = __ffs(bal) - 1;
        bal &= bal - 1;
        const int row = __shfl_sync(0xffffffffu, sv, b);
        T* dst = reinterpret_cast<T*>(const_cast<void*>(xr.p[(g + b) / El])) + (long long)row * d;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int v = v0 + q * 32 + lane;
          if (v < nvec) st_v4(dst + (long long)v * V, buf[q]);
        }
      }
    }
  }
}

// Exchange / GEMM overlap: arrival plan.  sprefix [E + 1]: prefix of this rank's
// counts in (local expert j, owner p) order (index j * W + p, global expert p * El + j) -- the
// order of the ordered send list; target [El] (cumulative over steps, wrap-safe): += the rows
// every source sends to my local expert j this step.
__global__ void ep2_arrival_plan_kernel(const int* __restrict__ counts_all, int W, int E, int me,
                                        int* __restrict__ sprefix, int* __restrict__ target) {
  const int El = E / W;
  __shared__ int s_c[128];              // this rank's counts in (j, p) order
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    const int j = i / W, p = i - j * W;
    s_c[i] = counts_all[(long long)me * E + p * El + j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < E; ++i) {
      sprefix[i] = acc;
      acc += s_c[i];
    }
    sprefix[E] = acc;
  }
  for (int j = threadIdx.x; j < El; j += blockDim.x) {
    int tot = 0;
    for (int q = 0; q < W; ++q) tot += counts_all[(long long)q * E + me * El + j];
    target[j] = (int)((unsigned)target[j] + (unsigned)tot);
  }
}

// token side copy pass in send-list order: block-chunks of kSendChunk entries, 32 per warp
// (x_t stored into its row on the owner), then one release add per (owner, local expert) of the
// chunk into the owner's arrival counters -- entries whose row was dropped (-1) count too, so the
// counters always reach the plan's targets.
constexpr int kSendChunk = 256;     // 8 warps x 32 entries
template <typename T>
__global__ void __launch_bounds__(256) ep2_copy_ordered_kernel(const T* __restrict__ x, const int* __restrict__ slot,
                                                               const int* __restrict__ send,
                                                               const int* __restrict__ sprefix, int d, int E, int El,
                                                               int W, const __grid_constant__ PeerTable xr,
                                                               const __grid_constant__ PeerTable arrive) {
  __shared__ int s_pref[129];
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_pref[i] = sprefix[i];
  __syncthreads();
  const int n = s_pref[E];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  auto idx_of = [&](int i) {          // largest idx with s_pref[idx] <= i
    int lo = 0, hi = E - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pref[mid] <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  for (int c0 = blockIdx.x * kSendChunk; c0 < n; c0 += gridDim.x * kSendChunk) {
    const int c1 = min(n, c0 + kSendChunk);
    // lane-parallel entry metadata (token, owner, row) of this warp's 32 entries, then the rows
    // four at a time with their loads in flight
    const int i = c0 + warp * 32 + lane;
    int tl = 0, pl = 0, rl = -1;
    if (i < c1) {
      const int idx = idx_of(i);
      const int j = idx / W;
      pl = idx - j * W;
      tl = send[i];
      rl = slot[(long long)tl * E + pl * El + j];
    }
    for (int b = 0; b < 32; b += 4) {
      int tt[4], rr[4], pp[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tt[k] = __shfl_sync(0xffffffffu, tl, b + k);
        rr[k] = __shfl_sync(0xffffffffu, rl, b + k);
        pp[k] = __shfl_sync(0xffffffffu, pl, b + k);
      }
      if (rr[0] < 0 && rr[1] < 0 && rr[2] < 0 && rr[3] < 0) continue;
      for (int v = lane; v < nvec; v += 32) {
        uint4 buf[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (rr[k] >= 0) buf[k] = ld_nc_v4(x + (long long)tt[k] * d + (long long)v * V);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (rr[k] >= 0)
            st_v4(reinterpret_cast<T*>(const_cast<void*>(xr.p[pp[k]])) + (long long)rr[k] * d + (long long)v * V,
                  buf[k]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int idx = idx_of(c0); idx < E && s_pref[idx] < c1; ++idx) {
        const int cnt = min(c1, s_pref[idx + 1]) - max(c0, s_pref[idx]);
        if (cnt <= 0) continue;
        const int j = idx / W, p = idx - j * W;
        int* a = reinterpret_cast<int*>(const_cast<void*>(arrive.p[p])) + j;
        asm volatile("red.release.sys.global.add.s32 [%0], %1;" ::"l"(a), "r"(cnt) : "memory");
      }
    }
    __syncthreads();
  }
}

// token side: y[t] = sum_{e asc} probs[t,e] e_out@(e / El)[slot[t,e]]
template <typename T, int QV>
__global__ void __launch_bounds__(256, 4) ep2_combine_kernel(const __grid_constant__ PeerTable eo,
                                                             const float* __restrict__ probs,
                                                             const int* __restrict__ slot, int T_, int d, int E, int El,
                                                             T* __restrict__ y) {
  constexpr int TPW = combine_tpw<QV>();          // as combine_kernel: both slot rows up front
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t0 = (blockIdx.x * 8 + warp) * TPW;
  if (t0 >= T_) return;
  int sv[TPW][4];
#pragma unroll
  for (int j = 0; j < TPW; ++j)
    if (t0 + j < T_) load_slot_row(slot + (long long)(t0 + j) * E, E, lane, sv[j]);
#pragma unroll
  for (int j = 0; j < TPW; ++j)
    if (t0 + j < T_)
      gather_sum_token_sv<T, true, float, QV, PeerRows<T>>(PeerRows<T>{&eo, probs + (long long)(t0 + j) * E, d, El},
                                                           sv[j], d, E, (const float*)nullptr,
                                                           y + (long long)(t0 + j) * d, lane);
}

// token side: dx[t] = dxg[t] + sum_{e asc} dx_perm@(e / El)[slot[t,e]]
template <typename T, typename TX, int QV>
__global__ void __launch_bounds__(256, 4) ep2_dispatch_bwd_kernel(const __grid_constant__ PeerTable dxp,
                                                                  const int* __restrict__ slot,
                                                                  const TX* dxg, int T_, int d, int E,
                                                                  int El, T* dx) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t = blockIdx.x * 8 + warp;
  if (t >= T_) return;
  gather_sum_token<T, false, TX, QV, PeerRows<T>>(PeerRows<T>{&dxp, nullptr, d, El}, slot + (long long)t * E, d, E,
                                                   dxg ? dxg + (long long)t * d : nullptr, dx + (long long)t * d, lane);
}

// ------------------------------------------------------------------ ep2 with token dedup ("ep2d")
// a token is sent ONCE to each GPU that owns any of its selected experts, and
// the owner pre-sums its local experts' contributions before the return trip.  Unique slot
// of token t of source rank s on every owner: u = s * T + t (fixed stride, no counts
// exchange).  Per owner: tokbuf [W*T, d] (x rows), urows [W*T, El] (the expert-side row of
// (u, local expert j), -1 if not selected: the token side writes the whole El-row for every
// owner each step), ruid [R_cap] (row -> u).  Token side: uslot [T, W] = u on owner q, or -1.

// token side rank pass (as dispatch_rank_kernel): my i-th token of expert e goes to row
// base[e] + i on rank e / El; slot <- that row; the row's metadata is stored at the owner.
// DEDUP (ep2d) also stores ruid at the owner, the token's urows rows on every owner (-1 for
// unselected experts) and its uslot row.
template <bool DEDUP>
__global__ void __launch_bounds__(kGateBT) ep2_rank_kernel(
    const float* __restrict__ probs, int* __restrict__ slot, int T_, int E, int El, int me, int W,
    const int* __restrict__ blk_base, const int* __restrict__ base, long long R_cap,
    const __grid_constant__ PeerTable rtok, const __grid_constant__ PeerTable rsrc,
    const __grid_constant__ PeerTable rgate, const __grid_constant__ PeerTable ruid,
    const __grid_constant__ PeerTable urows, int* __restrict__ uslot, int* __restrict__ send = nullptr,
    const int* __restrict__ sprefix = nullptr) {
  __shared__ unsigned s_bal[kGateBT / 32][128];
  __shared__ long long s_base[128];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int t = blockIdx.x * kGateBT + tid;
  const bool valid = t < T_;
  // the block's first row of every expert on its owner (as dispatch_rank_kernel)
  for (int e = tid; e < E; e += kGateBT) s_base[e] = (long long)base[e] + blk_base[(long long)e * gridDim.x + blockIdx.x];
  // 16 selection flags per thread in flight (16-byte loads when the rows allow), then 16 ballots
  const bool vec = (E & 3) == 0;
  unsigned selm[4] = {0u, 0u, 0u, 0u};              // this thread's selected experts (E <= 128)
  for (int e0 = 0; e0 < E; e0 += 16) {
    int v[16];
    if (vec && e0 + 16 <= E) {
      int4 q[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        q[i] = make_int4(-1, -1, -1, -1);
        if (valid) q[i] = *reinterpret_cast<const int4*>(slot + (long long)t * E + e0 + 4 * i);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) { v[4 * i] = q[i].x; v[4 * i + 1] = q[i].y; v[4 * i + 2] = q[i].z; v[4 * i + 3] = q[i].w; }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = (valid && e0 + j < E) ? slot[(long long)t * E + e0 + j] : -1;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const bool sel = v[j] >= 0 && e0 + j < E;
      const unsigned bal = __ballot_sync(0xffffffffu, sel);
      if (lane == 0 && e0 + j < E) s_bal[warp][e0 + j] = bal;
      if (sel) selm[(e0 + j) >> 5] |= 1u << ((e0 + j) & 31);
    }
  }
  __syncthreads();
  if (!valid) return;
  const unsigned lower = (1u << lane) - 1u;
  const long long u = (long long)me * T_ + t;
  if (!DEDUP) {
    // the selected experts only, ascending, up to 8 per batch with their gate loads in flight
    int word = 0;
    unsigned bits = selm[0];
    while (true) {
      int es[8], nb = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        while (bits == 0u && word < 3) bits = selm[++word];
        es[j] = -1;
        if (bits) {
          es[j] = word * 32 + __ffs(bits) - 1;
          bits &= bits - 1u;
          ++nb;
        }
      }
      if (nb == 0) break;
      float pg[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) pg[j] = es[j] >= 0 ? probs[(long long)t * E + es[j]] : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = es[j];
        if (e < 0) continue;
        const unsigned mine = s_bal[warp][e];
        int wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += __popc(s_bal[w][e]);
        const long long r = s_base[e] + wpre + __popc(mine & lower);
        int row = -1;
        if (r < R_cap) {
          const int p = e / El;
          row = (int)r;
          reinterpret_cast<int*>(const_cast<void*>(rtok.p[p]))[r] = t;
          reinterpret_cast<int*>(const_cast<void*>(rsrc.p[p]))[r] = me;
          reinterpret_cast<float*>(const_cast<void*>(rgate.p[p]))[r] = pg[j];
        }
        slot[(long long)t * E + e] = row;            // -1: dropped (MOE_ECAPACITY raised by the plan)
        // ordered send list (overlap mode): entry (e, local position r - base[e]) in (local expert,
        // owner) order, so the copy pass fills every owner's expert 0 first, then expert 1, ...
        if (send) send[sprefix[(e % El) * W + e / El] + (int)(r - base[e])] = t;
      }
      if (nb < 8) break;
    }
    return;
  }
  // dedup: every (token, local expert) entry of urows on every owner is written (the row or -1),
  // four contiguous entries per 16-byte store when El allows
  const bool v4 = (El & 3) == 0;
  for (int p = 0; p < W; ++p) {
    int* ur = reinterpret_cast<int*>(const_cast<void*>(urows.p[p])) + u * El;
    for (int j0 = 0; j0 < El; j0 += 4) {
      int rows4[4] = {-1, -1, -1, -1};
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = j0 + jj, e = p * El + j;
        if (j >= El) break;
        const unsigned mine = s_bal[warp][e];
        if (!((mine >> lane) & 1u)) continue;
        int wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += __popc(s_bal[w][e]);
        const long long r = s_base[e] + wpre + __popc(mine & lower);
        int row = -1;
        if (r < R_cap) {
          row = (int)r;
          reinterpret_cast<int*>(const_cast<void*>(rtok.p[p]))[r] = t;
          reinterpret_cast<int*>(const_cast<void*>(rsrc.p[p]))[r] = me;
          reinterpret_cast<float*>(const_cast<void*>(rgate.p[p]))[r] = probs[(long long)t * E + e];
          reinterpret_cast<int*>(const_cast<void*>(ruid.p[p]))[r] = (int)u;
        }
        slot[(long long)t * E + e] = row;          // -1: dropped (MOE_ECAPACITY raised by the plan)
        rows4[jj] = row;
      }
      if (v4) {
        *reinterpret_cast<int4*>(ur + j0) = make_int4(rows4[0], rows4[1], rows4[2], rows4[3]);
      } else {
        for (int jj = 0; jj < 4 && j0 + jj < El; ++jj) ur[j0 + jj] = rows4[jj];
      }
    }
  }
  if (DEDUP) {
    for (int p = 0; p < W; ++p) {
      bool any = false;
      for (int j = 0; j < El; ++j) any |= ((s_bal[warp][p * El + j] >> lane) & 1u) != 0;
      uslot[(long long)t * W + p] = any ? (int)u : -1;
    }
  }
}

// token side copy pass: x_t read once, stored once into tokbuf[u] of every owner it needs
template <typename T>
__global__ void __launch_bounds__(256) ep2d_copy_kernel(const T* __restrict__ x, const int* __restrict__ uslot, int T_,
                                                        int d, int W, const __grid_constant__ PeerTable tb) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int t = blockIdx.x * 8 + warp;
  if (t >= T_) return;
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  const int sv = lane < W ? uslot[(long long)t * W + lane] : -1;
  const unsigned bal0 = __ballot_sync(0xffffffffu, sv >= 0);
  const T* src = x + (long long)t * d;
  for (int v0 = 0; v0 < nvec; v0 += 32 * 4) {
    uint4 buf[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int v = v0 + q * 32 + lane;
      if (v < nvec) buf[q] = ld_nc_v4(src + (long long)v * V);
    }
    unsigned bal = bal0;
    while (bal) {
      const int p = __ffs(bal) - 1;
      bal &= bal - 1;
      const long long u = __shfl_sync(0xffffffffu, sv, p);
      T* dst = reinterpret_cast<T*>(const_cast<void*>(tb.p[p])) + u * d;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int v = v0 + q * 32 + lane;
        if (v < nvec) st_v4(dst + (long long)v * V, buf[q]);
      }
    }
  }
}

// expert side: x_recv[r] = tokbuf[ruid[r]] for the routed rows (pads were zeroed by ep2_prepare)
// Pad rows get ruid = -1: the combine backward takes ruid as its row -> token map and must
// see them as pads (a stale id would pull a dy row into a zero-gate pad row).
template <typename T>
__global__ void __launch_bounds__(256) ep2d_permute_kernel(const T* __restrict__ tokbuf, const int* __restrict__ rtok,
                                                           int* __restrict__ ruid, const int* __restrict__ off,
                                                           int El, int d, long long R_cap, T* __restrict__ x_recv) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long r = (long long)blockIdx.x * 8 + warp;
  if (r >= min((long long)off[El], R_cap)) return;
  if (rtok[r] < 0) {
    if (lane == 0) ruid[r] = -1;
    return;
  }
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  const T* src = tokbuf + (long long)ruid[r] * d;
  T* dst = x_recv + r * d;
  for (int v0 = 0; v0 < nvec; v0 += 32 * 4) {
    uint4 buf[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int v = v0 + q * 32 + lane;
      if (v < nvec) buf[q] = ld_nc_v4(src + (long long)v * V);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int v = v0 + q * 32 + lane;
      if (v < nvec) st_v4(dst + (long long)v * V, buf[q]);
    }
  }
}

// expert side pre-sum per unique token u: out[u] = sum_{j asc} (gate[row] *) rows[row],
// row = urows[u][j] >= 0 (local experts in ascending order); u with no row is skipped
template <typename T, bool WEIGHTED, int QV>
__global__ void __launch_bounds__(256, 4) ep2d_presum_kernel(const T* __restrict__ rows, const float* __restrict__ gate,
                                                             const int* __restrict__ urows, long long n_u, int El, int d,
                                                             T* __restrict__ out) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long u = (long long)blockIdx.x * 8 + warp;
  if (u >= n_u) return;
  const int* ur = urows + u * El;
  bool any = false;
  for (int j = lane; j < El; j += 32) any |= ur[j] >= 0;
  if (!__any_sync(0xffffffffu, any)) return;
  gather_sum_token<T, WEIGHTED, float, QV>(LocalRows<T>{rows, gate, d}, ur, d, El, nullptr, out + u * d, lane);
}

// expert side: dyu[u] = dy@s[t] for every unique token u = s * T + t routed here (one NVLink
// read per (token, owner) instead of one per selected expert)
template <typename T>
__global__ void __launch_bounds__(256) ep2d_gather_dy_kernel(const __grid_constant__ PeerTable dyp,
                                                             const int* __restrict__ urows, int T_, int W, int El,
                                                             int d, T* __restrict__ dyu) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long u = (long long)blockIdx.x * 8 + warp;
  if (u >= (long long)W * T_) return;
  const int* ur = urows + u * El;
  bool any = false;
  for (int j = lane; j < El; j += 32) any |= ur[j] >= 0;
  if (!__any_sync(0xffffffffu, any)) return;
  const int s = (int)(u / T_), t = (int)(u - (long long)s * T_);
  constexpr int V = Vec16<T>::N;
  const int nvec = d / V;
  const T* src = reinterpret_cast<const T*>(dyp.p[s]) + (long long)t * d;
  T* dst = dyu + u * d;
  for (int v0 = 0; v0 < nvec; v0 += 32 * 4) {
    uint4 buf[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int v = v0 + q * 32 + lane;
      if (v < nvec) buf[q] = ld_nc_v4(src + (long long)v * V);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int v = v0 + q * 32 + lane;
      if (v < nvec) st_v4(dst + (long long)v * V, buf[q]);
    }
  }
}

}  // namespace

cudaError_t launch_spawn(const moe_ctx* c, const void* W1s, const void* b1s, const void* W2s, const void* b2s,
                         const uint32_t* M1, const uint32_t* M2, void* W1, void* b1, void* W2, void* b2,
                         cudaStream_t s) {
  if (c->dtype == 1) return spawn_typed<bf16>(c, W1s, b1s, W2s, b2s, M1, M2, W1, b1, W2, b2, s);
  return spawn_typed<float>(c, W1s, b1s, W2s, b2s, M1, M2, W1, b1, W2, b2, s);
}

cudaError_t launch_dispatch(const moe_ctx* c, const void* x, const float* probs, int32_t* slot,
                            const int32_t* /*counts*/, void* x_perm, int32_t* row_token, float* row_gate,
                            int32_t* offsets, int64_t R_cap, int32_t* R_out, cudaStream_t s) {
  launch_dispatch_scan(c, offsets, R_out, R_cap, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || c->nblk == 0) return e;
  if (c->dtype == 1) {
    dispatch_rank_kernel<bf16><<<c->nblk, kGateBT, 0, s>>>(probs, slot, c->T, c->d, c->E, c->blk_base, offsets, c->tot,
                                                          (bf16*)x_perm, row_token, row_gate, R_cap), count_launch();
    dispatch_copy_kernel<bf16><<<(c->T + 7) / 8, 256, 0, s>>>((const bf16*)x, slot, c->T, c->d, c->E, (bf16*)x_perm),
        count_launch();
  } else {
    dispatch_rank_kernel<float><<<c->nblk, kGateBT, 0, s>>>(probs, slot, c->T, c->d, c->E, c->blk_base, offsets,
                                                           c->tot, (float*)x_perm, row_token, row_gate, R_cap),
        count_launch();
    dispatch_copy_kernel<float><<<(c->T + 7) / 8, 256, 0, s>>>((const float*)x, slot, c->T, c->d, c->E,
                                                               (float*)x_perm), count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_combine(const moe_ctx* c, const void* e_out, const float* row_gate, const int32_t* slot,
                           void* y, cudaStream_t s) {
  if (c->T == 0) return cudaSuccess;
#define MOE_QV_DISPATCH(qv, ...) \
  switch (qv) { case 1: { constexpr int QV = 1; __VA_ARGS__; } break; case 2: { constexpr int QV = 2; __VA_ARGS__; } break; \
                case 3: { constexpr int QV = 3; __VA_ARGS__; } break; default: { constexpr int QV = 4; __VA_ARGS__; } }
  if (c->dtype == 1) {
    MOE_QV_DISPATCH(pass_vectors(c->d, 8), combine_kernel<bf16, QV><<<(c->T + 8 * combine_tpw<QV>() - 1) /
                                                                           (8 * combine_tpw<QV>()), 256, 0, s>>>(
        (const bf16*)e_out, row_gate, slot, c->T, c->d, c->E, (bf16*)y), count_launch())
  } else {
    MOE_QV_DISPATCH(pass_vectors(c->d, 4), combine_kernel<float, QV><<<(c->T + 8 * combine_tpw<QV>() - 1) /
                                                                            (8 * combine_tpw<QV>()), 256, 0, s>>>(
        (const float*)e_out, row_gate, slot, c->T, c->d, c->E, (float*)y), count_launch())
  }
  return cudaGetLastError();
}

template <typename T, int MAXV, bool COMPUTE = true, bool PEER = false>
static cudaError_t launch_cbc(moe_ctx* c, const void* dy, const void* e_out, const float* row_gate,
                              const int32_t* row_token, const int32_t* offsets, int64_t R_cap, void* d_eout,
                              float* dG_row, cudaStream_t s, const int32_t* row_src = nullptr,
                              const PeerTable* dyp = nullptr) {
  const size_t smem = cb_smem_bytes<MAXV>();         // >= the [8][d] fp32 block reduction
  auto k = combine_bwd_colsum_kernel<T, MAXV, COMPUTE, PEER>;
  PeerTable tab{};
  if (dyp) tab = *dyp;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<dim3(c->db2_S, c->E_local), 256, smem, s>>>((const T*)dy, (const T*)e_out, row_gate, row_token, offsets, c->d,
                                                 R_cap, c->db2_S, (T*)d_eout, dG_row, c->db2part, row_src, tab),
      count_launch();
  return cudaGetLastError();
}

// db2 partials (c->db2part) of an existing d_eout with the fused kernel's partition; false if
// d is too wide for it (the caller then uses the generic column sums).
static bool launch_db2_partials(moe_ctx* c, const void* d_eout, const int32_t* offsets, int64_t R_cap, cudaStream_t s,
                                cudaError_t* err) {
  const int V = c->dtype == 1 ? 8 : 4, nvec = c->d / V;
  if (R_cap == 0) { *err = cudaSuccess; return false; }
  if (c->dtype == 1) {
    if (nvec <= 32) { *err = launch_cbc<bf16, 1, false>(c, nullptr, nullptr, nullptr, nullptr, offsets, R_cap, (void*)d_eout, nullptr, s); return true; }
    if (nvec <= 64) { *err = launch_cbc<bf16, 2, false>(c, nullptr, nullptr, nullptr, nullptr, offsets, R_cap, (void*)d_eout, nullptr, s); return true; }
    if (nvec <= 96) { *err = launch_cbc<bf16, 3, false>(c, nullptr, nullptr, nullptr, nullptr, offsets, R_cap, (void*)d_eout, nullptr, s); return true; }
    if (nvec <= 128) { *err = launch_cbc<bf16, 4, false>(c, nullptr, nullptr, nullptr, nullptr, offsets, R_cap, (void*)d_eout, nullptr, s); return true; }
  } else {
    if (nvec <= 32) { *err = launch_cbc<float, 1, false>(c, nullptr, nullptr, nullptr, nullptr, offsets, R_cap, (void*)d_eout, nullptr, s); return true; }
    if (nvec <= 64) { *err = launch_cbc<float, 2, false>(c, nullptr, nullptr, nullptr, nullptr, offsets, R_cap, (void*)d_eout, nullptr, s); return true; }
  }
  return false;
}

// db2 from an existing d_eout (moe_expert_ffn_bwd): the same partition and fixed order as the
// partials the fused combine backward produces, so both routes give bit-identical db2
cudaError_t launch_db2(moe_ctx* c, const void* d_eout, const int32_t* offsets, int64_t R_cap, float* db2,
                       cudaStream_t s) {
  if (R_cap == 0) return cudaMemsetAsync(db2, 0, sizeof(float) * c->E_local * c->d, s);
  cudaError_t e = cudaSuccess;
  if (!launch_db2_partials(c, d_eout, offsets, R_cap, s, &e))
    return launch_colsum_grouped(d_eout, c->dtype, c->d, offsets, c->E_local, db2, c->colpart, s);
  if (e != cudaSuccess) return e;
  return launch_colsum_final(c->db2part, c->d, c->db2_S, c->E_local, db2, s);
}

// finish db2 from the partials the fused combine backward just wrote (same call)
static cudaError_t finish_db2(moe_ctx* c, cudaError_t e, float* db2, cudaStream_t s) {
  if (e != cudaSuccess || !db2) return e;
  return launch_colsum_final(c->db2part, c->d, c->db2_S, c->E_local, db2, s);
}

cudaError_t launch_combine_bwd(moe_ctx* c, const void* dy, const void* e_out, const float* row_gate,
                               const int32_t* row_token, const int32_t* offsets, int64_t R_cap, void* d_eout,
                               float* dG_row, float* db2, cudaStream_t s) {
  if (R_cap == 0) return db2 ? cudaMemsetAsync(db2, 0, sizeof(float) * c->E_local * c->d, s) : cudaSuccess;
  if (c->world == 1 && !c->comm && c->E_local == c->E) {
    // single rank: the fused kernel also sums the d_eout it stores into the db2 partials
    const int V = c->dtype == 1 ? 8 : 4, nvec = c->d / V;
    if (c->dtype == 1) {
      if (nvec <= 32) return finish_db2(c, launch_cbc<bf16, 1>(c, dy, e_out, row_gate, row_token, offsets, R_cap, d_eout, dG_row, s), db2, s);
      if (nvec <= 64) return finish_db2(c, launch_cbc<bf16, 2>(c, dy, e_out, row_gate, row_token, offsets, R_cap, d_eout, dG_row, s), db2, s);
      if (nvec <= 96) return finish_db2(c, launch_cbc<bf16, 3>(c, dy, e_out, row_gate, row_token, offsets, R_cap, d_eout, dG_row, s), db2, s);
      if (nvec <= 128) return finish_db2(c, launch_cbc<bf16, 4>(c, dy, e_out, row_gate, row_token, offsets, R_cap, d_eout, dG_row, s), db2, s);
    } else {
      if (nvec <= 32) return finish_db2(c, launch_cbc<float, 1>(c, dy, e_out, row_gate, row_token, offsets, R_cap, d_eout, dG_row, s), db2, s);
      if (nvec <= 64) return finish_db2(c, launch_cbc<float, 2>(c, dy, e_out, row_gate, row_token, offsets, R_cap, d_eout, dG_row, s), db2, s);
    }
  }
  const unsigned grid = (unsigned)((R_cap + 7) / 8);
  if (c->dtype == 1)
    combine_bwd_kernel<bf16><<<grid, 256, 0, s>>>((const bf16*)dy, (const bf16*)e_out, row_gate, row_token, offsets,
                                                  c->E, c->d, R_cap, (bf16*)d_eout, dG_row, nullptr, PeerTable{}),
        count_launch();
  else
    combine_bwd_kernel<float><<<grid, 256, 0, s>>>((const float*)dy, (const float*)e_out, row_gate, row_token,
                                                   offsets, c->E, c->d, R_cap, (float*)d_eout, dG_row, nullptr,
                                                   PeerTable{}), count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess && db2 ? launch_db2(c, d_eout, offsets, R_cap, db2, s) : e;
}

cudaError_t launch_dispatch_bwd(const moe_ctx* c, const void* dx_perm, const int32_t* slot, int accumulate,
                                void* dx, cudaStream_t s) {
  if (c->T == 0) return cudaSuccess;
  const unsigned grid = (c->T + 7) / 8;
  // accumulate: each warp loads its token's dx row (written by moe_dts_gate_bwd: dlogits W_g^T)
  // before it sums the selected dx_perm rows onto it and stores the row back
  if (c->dtype == 1)
    MOE_QV_DISPATCH(pass_vectors(c->d, 8), dispatch_bwd_kernel<bf16, bf16, QV><<<grid, 256, 0, s>>>((const bf16*)dx_perm, slot,
                                                         accumulate ? (const bf16*)dx : nullptr, c->T, c->d, c->E, (bf16*)dx), count_launch())
  else
    MOE_QV_DISPATCH(pass_vectors(c->d, 4), dispatch_bwd_kernel<float, float, QV><<<grid, 256, 0, s>>>((const float*)dx_perm, slot,
                                                           accumulate ? (const float*)dx : nullptr, c->T, c->d, c->E, (float*)dx), count_launch())
  return cudaGetLastError();
}

}  // namespace moe

namespace moe {

// ------------------------------------------------------------------ fused peer-memory EP launchers
cudaError_t launch_ep2_counts(const moe_ctx* c, const int32_t* counts, const PeerTable& all, cudaStream_t s) {
  const int n = c->world * c->E;
  ep2_counts_kernel<<<(n + 255) / 256, 256, 0, s>>>(counts, c->E, c->rank, c->world, all), count_launch();
  return cudaGetLastError();
}

cudaError_t launch_ep2_plan(const moe_ctx* c, const int32_t* counts_all, int64_t R_cap, int32_t* offsets_recv,
                            cudaStream_t s) {
  ep2_plan_kernel<<<1, 256, sizeof(long long) * c->E, s>>>(counts_all, c->world, c->E, c->rank, R_cap, c->ep_off,
                                                          c->ep_tot, c->ep2_base, c->flags), count_launch();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && offsets_recv)
    e = cudaMemcpyAsync(offsets_recv, c->ep_off, sizeof(int) * (c->E_local + 1), cudaMemcpyDeviceToDevice, s);
  return e;
}

cudaError_t launch_ep2_prepare(const moe_ctx* c, void* x_recv, int32_t* rtok, int32_t* rsrc, float* rgate,
                               int64_t R_cap, cudaStream_t s) {
  dim3 grid(64, c->E_local < 65535 ? c->E_local : 65535);
  if (c->dtype == 1)
    ep2_prepare_kernel<bf16><<<grid, 256, 0, s>>>((bf16*)x_recv, rtok, rsrc, rgate, c->ep_off, c->ep_tot, c->E_local,
                                                  c->d, R_cap), count_launch();
  else
    ep2_prepare_kernel<float><<<grid, 256, 0, s>>>((float*)x_recv, rtok, rsrc, rgate, c->ep_off, c->ep_tot, c->E_local,
                                                   c->d, R_cap), count_launch();
  return cudaGetLastError();
}

cudaError_t launch_ep2_arrival_plan(const moe_ctx* c, const int32_t* counts_all, int32_t* sprefix, int32_t* target,
                                    cudaStream_t s) {
  ep2_arrival_plan_kernel<<<1, 128, 0, s>>>(counts_all, c->world, c->E, c->rank, sprefix, target), count_launch();
  return cudaGetLastError();
}

cudaError_t launch_ep2_dispatch(const moe_ctx* c, const void* x, const float* probs, int32_t* slot, const PeerTable& xr,
                                const PeerTable& rtok, const PeerTable& rsrc, const PeerTable& rgate, int64_t R_cap,
                                cudaStream_t s, const int32_t* sprefix, int32_t* send, const PeerTable* arrive) {
  // per-block ranks (scan over this rank's token blocks; the local layout itself is not built)
  launch_dispatch_scan(c, c->ep2_scr, c->ep2_scr + c->E + 1, (long long)1 << 62, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || c->nblk == 0) return e;
  ep2_rank_kernel<false><<<c->nblk, kGateBT, 0, s>>>(probs, slot, c->T, c->E, c->E_local, c->rank, c->world,
                                                     c->blk_base, c->ep2_base, R_cap, rtok, rsrc, rgate, PeerTable{},
                                                     PeerTable{}, nullptr, send, sprefix), count_launch();
  if (send) {   // overlap mode: copy in send-list order with arrival counters
    const int grid = 4 * c->sm_count;
    if (c->dtype == 1)
      ep2_copy_ordered_kernel<bf16><<<grid, 256, 0, s>>>((const bf16*)x, slot, send, sprefix, c->d, c->E, c->E_local,
                                                         c->world, xr, *arrive), count_launch();
    else
      ep2_copy_ordered_kernel<float><<<grid, 256, 0, s>>>((const float*)x, slot, send, sprefix, c->d, c->E,
                                                          c->E_local, c->world, xr, *arrive), count_launch();
    return cudaGetLastError();
  }
  if (c->dtype == 1)
    ep2_copy_kernel<bf16><<<(c->T + 7) / 8, 256, 0, s>>>((const bf16*)x, slot, c->T, c->d, c->E, c->E_local, xr),
        count_launch();
  else
    ep2_copy_kernel<float><<<(c->T + 7) / 8, 256, 0, s>>>((const float*)x, slot, c->T, c->d, c->E, c->E_local, xr),
        count_launch();
  return cudaGetLastError();
}

cudaError_t launch_ep2_combine(const moe_ctx* c, const PeerTable& eo, const float* probs, const int32_t* slot, void* y,
                               cudaStream_t s) {
  if (c->T == 0) return cudaSuccess;
  if (c->dtype == 1) {
    MOE_QV_DISPATCH(pass_vectors(c->d, 8), ep2_combine_kernel<bf16, QV><<<(c->T + 8 * combine_tpw<QV>() - 1) /
                                                                               (8 * combine_tpw<QV>()), 256, 0, s>>>(
        eo, probs, slot, c->T, c->d, c->E, c->E_local, (bf16*)y), count_launch())
  } else {
    MOE_QV_DISPATCH(pass_vectors(c->d, 4), ep2_combine_kernel<float, QV><<<(c->T + 8 * combine_tpw<QV>() - 1) /
                                                                                (8 * combine_tpw<QV>()), 256, 0, s>>>(
        eo, probs, slot, c->T, c->d, c->E, c->E_local, (float*)y), count_launch())
  }
  return cudaGetLastError();
}

bool ep2_width_ok(const moe_ctx* c) {
  const int V = c->dtype == 1 ? 8 : 4, nvec = c->d / V;
  return c->dtype == 1 ? nvec <= 128 : nvec <= 64;
}

cudaError_t launch_ep2_combine_bwd(moe_ctx* c, const PeerTable& dyp, const void* e_out, const float* rgate,
                                   const int32_t* rtok, const int32_t* rsrc, const int32_t* offsets, int64_t R_cap,
                                   void* d_eout, float* dG_row, float* db2, cudaStream_t s) {
  if (R_cap == 0) return db2 ? cudaMemsetAsync(db2, 0, sizeof(float) * c->E_local * c->d, s) : cudaSuccess;
  const int V = c->dtype == 1 ? 8 : 4, nvec = c->d / V;
  cudaError_t e;
  if (!ep2_width_ok(c)) {
    // rows wider than the fused kernel's register budget: warp per row (dy through the peer
    // pointers), then db2 from the stored d_eout
    const unsigned grid = (unsigned)((R_cap + 7) / 8);
    if (c->dtype == 1)
      combine_bwd_kernel<bf16, true><<<grid, 256, 0, s>>>(nullptr, (const bf16*)e_out, rgate, rtok, offsets, c->E_local,
                                                          c->d, R_cap, (bf16*)d_eout, dG_row, rsrc, dyp), count_launch();
    else
      combine_bwd_kernel<float, true><<<grid, 256, 0, s>>>(nullptr, (const float*)e_out, rgate, rtok, offsets,
                                                           c->E_local, c->d, R_cap, (float*)d_eout, dG_row, rsrc, dyp),
          count_launch();
    e = cudaGetLastError();
    return e == cudaSuccess && db2 ? launch_db2(c, d_eout, offsets, R_cap, db2, s) : e;
  }
  if (c->dtype == 1) {
    if (nvec <= 32) e = launch_cbc<bf16, 1, true, true>(c, nullptr, e_out, rgate, rtok, offsets, R_cap, d_eout, dG_row, s, rsrc, &dyp);
    else if (nvec <= 64) e = launch_cbc<bf16, 2, true, true>(c, nullptr, e_out, rgate, rtok, offsets, R_cap, d_eout, dG_row, s, rsrc, &dyp);
    else if (nvec <= 96) e = launch_cbc<bf16, 3, true, true>(c, nullptr, e_out, rgate, rtok, offsets, R_cap, d_eout, dG_row, s, rsrc, &dyp);
    else e = launch_cbc<bf16, 4, true, true>(c, nullptr, e_out, rgate, rtok, offsets, R_cap, d_eout, dG_row, s, rsrc, &dyp);
  } else if (nvec <= 32) {
    e = launch_cbc<float, 1, true, true>(c, nullptr, e_out, rgate, rtok, offsets, R_cap, d_eout, dG_row, s, rsrc, &dyp);
  } else {
    e = launch_cbc<float, 2, true, true>(c, nullptr, e_out, rgate, rtok, offsets, R_cap, d_eout, dG_row, s, rsrc, &dyp);
  }
  return finish_db2(c, e, db2, s);
}

cudaError_t launch_ep2_dispatch_bwd(const moe_ctx* c, const PeerTable& dxp, const int32_t* slot, int accumulate,
                                    void* dx, cudaStream_t s, int slot_cols, int cols_per_rank) {
  if (c->T == 0) return cudaSuccess;
  const int SE = slot_cols > 0 ? slot_cols : c->E, SEl = cols_per_rank > 0 ? cols_per_rank : c->E_local;
  const unsigned grid = (c->T + 7) / 8;
  if (c->dtype == 1) {
    MOE_QV_DISPATCH(pass_vectors(c->d, 8), ep2_dispatch_bwd_kernel<bf16, bf16, QV><<<grid, 256, 0, s>>>(
        dxp, slot, accumulate ? (const bf16*)dx : nullptr, c->T, c->d, SE, SEl, (bf16*)dx), count_launch())
  } else {
    MOE_QV_DISPATCH(pass_vectors(c->d, 4), ep2_dispatch_bwd_kernel<float, float, QV><<<grid, 256, 0, s>>>(
        dxp, slot, accumulate ? (const float*)dx : nullptr, c->T, c->d, SE, SEl, (float*)dx), count_launch())
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ ep2 with token dedup
cudaError_t launch_ep2d_dispatch(const moe_ctx* c, const void* x, const float* probs, int32_t* slot, int32_t* uslot,
                                 const PeerTable& tb, const PeerTable& urows, const PeerTable& rtok,
                                 const PeerTable& rsrc, const PeerTable& rgate, const PeerTable& ruid, int64_t R_cap,
                                 cudaStream_t s) {
  launch_dispatch_scan(c, c->ep2_scr, c->ep2_scr + c->E + 1, (long long)1 << 62, s);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || c->nblk == 0) return e;
  ep2_rank_kernel<true><<<c->nblk, kGateBT, 0, s>>>(probs, slot, c->T, c->E, c->E_local, c->rank, c->world,
                                                    c->blk_base, c->ep2_base, R_cap, rtok, rsrc, rgate, ruid, urows,
                                                    uslot), count_launch();
  if (c->dtype == 1)
    ep2d_copy_kernel<bf16><<<(c->T + 7) / 8, 256, 0, s>>>((const bf16*)x, uslot, c->T, c->d, c->world, tb),
        count_launch();
  else
    ep2d_copy_kernel<float><<<(c->T + 7) / 8, 256, 0, s>>>((const float*)x, uslot, c->T, c->d, c->world, tb),
        count_launch();
  return cudaGetLastError();
}

cudaError_t launch_ep2d_permute(const moe_ctx* c, const void* tokbuf, const int32_t* rtok, int32_t* ruid,
                                int64_t R_cap, void* x_recv, cudaStream_t s) {
  if (R_cap == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((R_cap + 7) / 8);
  if (c->dtype == 1)
    ep2d_permute_kernel<bf16><<<grid, 256, 0, s>>>((const bf16*)tokbuf, rtok, ruid, c->ep_off, c->E_local, c->d,
                                                   R_cap, (bf16*)x_recv), count_launch();
  else
    ep2d_permute_kernel<float><<<grid, 256, 0, s>>>((const float*)tokbuf, rtok, ruid, c->ep_off, c->E_local, c->d,
                                                    R_cap, (float*)x_recv), count_launch();
  return cudaGetLastError();
}

cudaError_t launch_ep2d_presum(const moe_ctx* c, const void* rows, const float* gate, const int32_t* urows, void* out,
                               cudaStream_t s) {
  const long long n_u = (long long)c->world * c->T;
  if (n_u == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((n_u + 7) / 8);
  const int El = c->E_local;
  if (c->dtype == 1) {
    if (gate) {
      MOE_QV_DISPATCH(pass_vectors(c->d, 8), ep2d_presum_kernel<bf16, true, QV><<<grid, 256, 0, s>>>(
          (const bf16*)rows, gate, urows, n_u, El, c->d, (bf16*)out), count_launch())
    } else {
      MOE_QV_DISPATCH(pass_vectors(c->d, 8), ep2d_presum_kernel<bf16, false, QV><<<grid, 256, 0, s>>>(
          (const bf16*)rows, gate, urows, n_u, El, c->d, (bf16*)out), count_launch())
    }
  } else {
    if (gate) {
      MOE_QV_DISPATCH(pass_vectors(c->d, 4), ep2d_presum_kernel<float, true, QV><<<grid, 256, 0, s>>>(
          (const float*)rows, gate, urows, n_u, El, c->d, (float*)out), count_launch())
    } else {
      MOE_QV_DISPATCH(pass_vectors(c->d, 4), ep2d_presum_kernel<float, false, QV><<<grid, 256, 0, s>>>(
          (const float*)rows, gate, urows, n_u, El, c->d, (float*)out), count_launch())
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_ep2d_gather_dy(const moe_ctx* c, const PeerTable& dyp, const int32_t* urows, void* dyu,
                                  cudaStream_t s) {
  const long long n_u = (long long)c->world * c->T;
  if (n_u == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((n_u + 7) / 8);
  if (c->dtype == 1)
    ep2d_gather_dy_kernel<bf16><<<grid, 256, 0, s>>>(dyp, urows, c->T, c->world, c->E_local, c->d, (bf16*)dyu),
        count_launch();
  else
    ep2d_gather_dy_kernel<float><<<grid, 256, 0, s>>>(dyp, urows, c->T, c->world, c->E_local, c->d, (float*)dyu),
        count_launch();
  return cudaGetLastError();
}

// token side: y[t] = sum_{q asc} ysum@q[uslot[t, q]] (the owners' pre-summed rows, unweighted)
cudaError_t launch_ep2d_combine(const moe_ctx* c, const PeerTable& ys, const int32_t* uslot, void* y, cudaStream_t s) {
  if (c->T == 0) return cudaSuccess;
  const unsigned grid = (c->T + 7) / 8;
  if (c->dtype == 1) {
    MOE_QV_DISPATCH(pass_vectors(c->d, 8), ep2_dispatch_bwd_kernel<bf16, float, QV><<<grid, 256, 0, s>>>(
        ys, uslot, nullptr, c->T, c->d, c->world, 1, (bf16*)y), count_launch())
  } else {
    MOE_QV_DISPATCH(pass_vectors(c->d, 4), ep2_dispatch_bwd_kernel<float, float, QV><<<grid, 256, 0, s>>>(
        ys, uslot, nullptr, c->T, c->d, c->world, 1, (float*)y), count_launch())
  }
  return cudaGetLastError();
}

// expert side combine backward with dy from the local dyu (row_token = ruid): the fused
// d_eout / dG / db2-partials kernel of the single-rank path
cudaError_t launch_ep2d_combine_bwd(moe_ctx* c, const void* dyu, const void* e_out, const float* rgate,
                                    const int32_t* ruid, const int32_t* offsets, int64_t R_cap, void* d_eout,
                                    float* dG_row, float* db2, cudaStream_t s) {
  if (R_cap == 0) return db2 ? cudaMemsetAsync(db2, 0, sizeof(float) * c->E_local * c->d, s) : cudaSuccess;
  const int V = c->dtype == 1 ? 8 : 4, nvec = c->d / V;
  cudaError_t e;
  if (!ep2_width_ok(c)) {
    // rows wider than the fused kernel's register budget: warp per row, then db2 from d_eout
    const unsigned grid = (unsigned)((R_cap + 7) / 8);
    if (c->dtype == 1)
      combine_bwd_kernel<bf16><<<grid, 256, 0, s>>>((const bf16*)dyu, (const bf16*)e_out, rgate, ruid, offsets,
                                                    c->E_local, c->d, R_cap, (bf16*)d_eout, dG_row, nullptr,
                                                    PeerTable{}), count_launch();
    else
      combine_bwd_kernel<float><<<grid, 256, 0, s>>>((const float*)dyu, (const float*)e_out, rgate, ruid, offsets,
                                                     c->E_local, c->d, R_cap, (float*)d_eout, dG_row, nullptr,
                                                     PeerTable{}), count_launch();
    e = cudaGetLastError();
    return e == cudaSuccess && db2 ? launch_db2(c, d_eout, offsets, R_cap, db2, s) : e;
  }
  if (c->dtype == 1) {
    if (nvec <= 32) e = launch_cbc<bf16, 1>(c, dyu, e_out, rgate, ruid, offsets, R_cap, d_eout, dG_row, s);
    else if (nvec <= 64) e = launch_cbc<bf16, 2>(c, dyu, e_out, rgate, ruid, offsets, R_cap, d_eout, dG_row, s);
    else if (nvec <= 96) e = launch_cbc<bf16, 3>(c, dyu, e_out, rgate, ruid, offsets, R_cap, d_eout, dG_row, s);
    else e = launch_cbc<bf16, 4>(c, dyu, e_out, rgate, ruid, offsets, R_cap, d_eout, dG_row, s);
  } else if (nvec <= 32) {
    e = launch_cbc<float, 1>(c, dyu, e_out, rgate, ruid, offsets, R_cap, d_eout, dG_row, s);
  } else {
    e = launch_cbc<float, 2>(c, dyu, e_out, rgate, ruid, offsets, R_cap, d_eout, dG_row, s);
  }
  return finish_db2(c, e, db2, s);
}

}  // namespace moe
