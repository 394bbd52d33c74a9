// ep.cu -- expert parallelism (EP, GShard-style): experts split E/W per rank,
// tokens data-parallel.  The exchange plan is pure host arithmetic on the gathered
// per-(rank, expert) counts; the row exchanges are grouped ncclSend/ncclRecv over
// NVLink/NVSwitch, one message per (peer, local expert) segment, written straight into
// the receiver's expert-major, 128-row-aligned layout (no re-layout pass).
//
//   token side  ("send" layout): moe_dispatch's global-expert-major layout, offsets_send
//   expert side ("recv" layout): local expert j holds the rows of every source rank q in
//                                ascending q (= ascending global token index), 128-aligned
//
// Multi-node: ep_build_hier / ep_exchange_hier route the inter-node rows through one relay
// GPU per (node, peer node), one inter-node message per ordered node pair (NEXT #4,
// P:405-408), landing in the same recv / send layouts.
#include <string.h>

#include <vector>

#include "common.cuh"
#include "internal.h"
#include "ep.h"

#ifdef MOE_HAVE_NCCL
#include <nccl.h>
#endif

namespace moe {

static inline long long align_rows(long long v) { return (v + kRowAlign - 1) / kRowAlign * kRowAlign; }

// counts_all[q * E + e] = number of rank q's tokens routed to global expert e.
void ep_build_plan(EpPlan& P, const int* counts_all, int W, int E, int rank) {
  P = EpPlan();
  P.W = W; P.E = E; P.El = E / W; P.rank = rank;
  const int El = P.El;
  P.offsets_send.assign(E + 1, 0);
  for (int e = 0; e < E; ++e)
    P.offsets_send[e + 1] = (int)(P.offsets_send[e] + align_rows(counts_all[(long long)rank * E + e]));
  P.R_send = P.offsets_send[E];
  P.offsets_recv.assign(El + 1, 0);
  P.recv_tot.assign(El, 0);
  for (int j = 0; j < El; ++j) {
    long long tot = 0;
    for (int q = 0; q < W; ++q) tot += counts_all[(long long)q * E + rank * El + j];
    P.recv_tot[j] = (int)tot;
    P.offsets_recv[j + 1] = (int)(P.offsets_recv[j] + align_rows(tot));
  }
  P.R_recv = P.offsets_recv[El];
  // sends: to peer p, its local experts in ascending order
  for (int p = 0; p < W; ++p)
    for (int j = 0; j < El; ++j) {
      const int e = p * El + j;
      const int n = counts_all[(long long)rank * E + e];
      if (n > 0) {
        P.s_peer.push_back(p);
        P.s_rows.push_back(n);
        P.s_src.push_back(P.offsets_send[e]);
      }
    }
  // recvs: from peer q, my local experts in ascending order (matches q's send order)
  for (int q = 0; q < W; ++q)
    for (int j = 0; j < El; ++j) {
      const int e = rank * El + j;
      const int n = counts_all[(long long)q * E + e];
      if (n > 0) {
        long long before = 0;
        for (int q2 = 0; q2 < q; ++q2) before += counts_all[(long long)q2 * E + e];
        P.r_peer.push_back(q);
        P.r_rows.push_back(n);
        P.r_dst.push_back(P.offsets_recv[j] + before);
      }
    }
}

// ------------------------------------------------------------------ hierarchical plan
// Nodes of G consecutive ranks.  Rows from node A to node B != A travel
//   phase 0: source q (in A) -> relay(A, B), gathered in stage_out ordered (p in B, j, q in A);
//   phase 1: relay(A, B) -> relay(B, A), ONE message per ordered node pair (G^2 pair payloads
//            aggregated, the paper's "#GPU^2 times larger" message), into stage_in;
//   phase 2: relay(B, A) -> destination p (in B), one segment per local expert j, written
//            straight into p's expert-major recv layout (the rows of the sources q in A are
//            contiguous there because A's ranks are consecutive).
// Same-node rows go directly in phase 0.  The combine runs the same messages reversed.
void ep_build_hier(EpHier& H, const int* counts_all, int W, int E, int rank, int G,
                   const std::vector<int>& offsets_send_me) {
  H = EpHier();
  H.G = G;
  H.N = W / G;
  const int N = H.N, El = E / W, A = rank / G, l = rank % G;
  auto cnt = [&](int q, int e) { return (long long)counts_all[(long long)q * E + e]; };
  // recv-layout offsets of (destination p = me) expert j, rows from source q onwards
  std::vector<long long> off_recv(El + 1, 0);
  for (int j = 0; j < El; ++j) {
    long long tot = 0;
    for (int q = 0; q < W; ++q) tot += cnt(q, rank * El + j);
    off_recv[j + 1] = off_recv[j] + align_rows(tot);
  }
  auto recv_row = [&](int j, int q_first) {
    long long r = off_recv[j];
    for (int q = 0; q < q_first; ++q) r += cnt(q, rank * El + j);
    return r;
  };
  // ---- stage_out (I relay for the remote nodes B with B % G == l): blocks ordered by B,
  //      inside (p in B, j, q in A)
  std::vector<long long> out_base(N, -1), out_len(N, 0);
  long long so = 0;
  for (int B = 0; B < N; ++B) {
    if (B == A || B % G != l) continue;
    out_base[B] = so;
    for (int p = B * G; p < (B + 1) * G; ++p)
      for (int j = 0; j < El; ++j)
        for (int q = A * G; q < (A + 1) * G; ++q) out_len[B] += cnt(q, p * El + j);
    so += out_len[B];
  }
  H.stage_out = so;
  // ---- stage_in (I relay for the source nodes A' with A' % G == l): blocks ordered by A',
  //      inside (p in A, j, q in A')
  std::vector<long long> in_base(N, -1), in_len(N, 0);
  long long si = 0;
  for (int Ap = 0; Ap < N; ++Ap) {
    if (Ap == A || Ap % G != l) continue;
    in_base[Ap] = si;
    for (int p = A * G; p < (A + 1) * G; ++p)
      for (int j = 0; j < El; ++j)
        for (int q = Ap * G; q < (Ap + 1) * G; ++q) in_len[Ap] += cnt(q, p * El + j);
    si += in_len[Ap];
  }
  H.stage_in = si;
  // ---- phase 0 sends (source = me), peers of my node in ascending rank: direct segments to
  //      the peer's own experts, then the segments the peer relays (B asc, p asc, j asc)
  for (int r = A * G; r < (A + 1) * G; ++r) {
    for (int j = 0; j < El; ++j) {
      const int e = r * El + j;
      const long long n = cnt(rank, e);
      if (n > 0) H.snd[0].push_back({r, 0, offsets_send_me[e], (int)n});
    }
    for (int B = 0; B < N; ++B) {
      if (B == A || ep_relay(A, B, G) != r) continue;
      for (int p = B * G; p < (B + 1) * G; ++p)
        for (int j = 0; j < El; ++j) {
          const int e = p * El + j;
          const long long n = cnt(rank, e);
          if (n > 0) H.snd[0].push_back({r, 0, offsets_send_me[e], (int)n});
        }
    }
  }
  // ---- phase 0 receives (in the same per-peer order): direct rows of my experts into the
  //      recv layout, then (if I relay) the gathered segments into stage_out
  for (int q = A * G; q < (A + 1) * G; ++q) {
    for (int j = 0; j < El; ++j) {
      const long long n = cnt(q, rank * El + j);
      if (n > 0) H.rcv[0].push_back({q, 1, recv_row(j, q), (int)n});
    }
    for (int B = 0; B < N; ++B) {
      if (B == A || B % G != l) continue;
      long long pos = out_base[B];
      for (int p = B * G; p < (B + 1) * G; ++p)
        for (int j = 0; j < El; ++j)
          for (int q2 = A * G; q2 < (A + 1) * G; ++q2) {
            const long long n = cnt(q2, p * El + j);
            if (q2 == q && n > 0) H.rcv[0].push_back({q, 2, pos, (int)n});
            pos += n;
          }
    }
  }
  // ---- phase 1: relay <-> relay, one message per ordered node pair
  for (int B = 0; B < N; ++B)
    if (B != A && B % G == l && out_len[B] > 0) H.snd[1].push_back({ep_relay(B, A, G), 2, out_base[B], (int)out_len[B]});
  for (int Ap = 0; Ap < N; ++Ap)
    if (Ap != A && Ap % G == l && in_len[Ap] > 0) H.rcv[1].push_back({ep_relay(Ap, A, G), 3, in_base[Ap], (int)in_len[Ap]});
  // ---- phase 2 sends (I relay the source nodes A' % G == l): to each p of my node, per
  //      (A' asc, j asc) the contiguous rows of A''s sources
  for (int p = A * G; p < (A + 1) * G; ++p) {
    for (int Ap = 0; Ap < N; ++Ap) {
      if (Ap == A || Ap % G != l) continue;
      long long pos = in_base[Ap];
      for (int p2 = A * G; p2 < (A + 1) * G; ++p2)
        for (int j = 0; j < El; ++j) {
          long long n = 0;
          for (int q = Ap * G; q < (Ap + 1) * G; ++q) n += cnt(q, p2 * El + j);
          if (p2 == p && n > 0) H.snd[2].push_back({p, 3, pos, (int)n});
          pos += n;
        }
    }
  }
  // ---- phase 2 receives (destination = me): from relay(A, A') for every remote node A'
  for (int Ap = 0; Ap < N; ++Ap) {
    if (Ap == A) continue;
    const int r = ep_relay(A, Ap, G);
    for (int j = 0; j < El; ++j) {
      long long n = 0;
      for (int q = Ap * G; q < (Ap + 1) * G; ++q) n += cnt(q, rank * El + j);
      if (n > 0) H.rcv[2].push_back({r, 1, recv_row(j, Ap * G), (int)n});
    }
  }
}

namespace {

// zero the pad rows [offsets[j] + tot[j], offsets[j+1]) of a recv-layout buffer
template <typename T>
__global__ void zero_pads_kernel(T* __restrict__ buf, const int* __restrict__ offsets, const int* __restrict__ tot,
                                 int El, int width) {
  const int j = blockIdx.y;
  if (j >= El) return;
  const long long r0 = (long long)offsets[j] + tot[j], r1 = offsets[j + 1];
  constexpr int V = Vec16<T>::N;
  const int nvec = width / V;
  for (long long r = r0 + blockIdx.x; r < r1; r += gridDim.x)
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) st_v4(buf + r * width + (long long)v * V, make_uint4(0, 0, 0, 0));
}

}  // namespace

cudaError_t launch_zero_pads(const moe_ctx* c, void* buf, const int* offsets_dev, const int* tot_dev, int width,
                             cudaStream_t s) {
  dim3 grid(128, c->E_local);
  if (c->dtype == 1)
    zero_pads_kernel<bf16><<<grid, 128, 0, s>>>((bf16*)buf, offsets_dev, tot_dev, c->E_local, width), count_launch();
  else
    zero_pads_kernel<float><<<grid, 128, 0, s>>>((float*)buf, offsets_dev, tot_dev, c->E_local, width), count_launch();
  return cudaGetLastError();
}

#ifdef MOE_HAVE_NCCL
ncclResult_t ep_exchange_hier(const moe_ctx* c, const EpPlan& P, const void* src, void* dst, void* stage, int width,
                              int direction, cudaStream_t s) {
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(c->comm);
  const size_t row_bytes = (size_t)width * (c->dtype == 1 ? 2 : 4);
  char* bufs[4];
  bufs[0] = const_cast<char*>(reinterpret_cast<const char*>(direction == 0 ? src : dst));   // send layout
  bufs[1] = const_cast<char*>(reinterpret_cast<const char*>(direction == 0 ? dst : src));   // recv layout
  bufs[2] = reinterpret_cast<char*>(stage);
  bufs[3] = bufs[2] ? bufs[2] + P.H.stage_out * row_bytes : nullptr;
  for (int k = 0; k < 3; ++k) {
    const int ph = direction == 0 ? k : 2 - k;
    // dispatch posts the phase's sends as sends; the combine runs every message backwards
    const std::vector<EpMsg>& as_send = direction == 0 ? P.H.snd[ph] : P.H.rcv[ph];
    const std::vector<EpMsg>& as_recv = direction == 0 ? P.H.rcv[ph] : P.H.snd[ph];
    if (as_send.empty() && as_recv.empty()) continue;
    ncclResult_t r = ncclGroupStart();
    if (r != ncclSuccess) return r;
    for (size_t i = 0; i < as_send.size() && r == ncclSuccess; ++i) {
      const EpMsg& m = as_send[i];
      r = ncclSend(bufs[m.buf] + m.row * row_bytes, (size_t)m.rows * row_bytes, ncclInt8, m.peer, comm, s);
    }
    for (size_t i = 0; i < as_recv.size() && r == ncclSuccess; ++i) {
      const EpMsg& m = as_recv[i];
      r = ncclRecv(bufs[m.buf] + m.row * row_bytes, (size_t)m.rows * row_bytes, ncclInt8, m.peer, comm, s);
    }
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return r;
    if (r2 != ncclSuccess) return r2;
  }
  return ncclSuccess;
}

// direction 0: send layout -> recv layout (dispatch);  1: recv -> send (combine)
ncclResult_t ep_exchange(const moe_ctx* c, const EpPlan& P, const void* src, void* dst, int width, int direction,
                         cudaStream_t s) {
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(c->comm);
  const size_t esz = c->dtype == 1 ? 2 : 4;
  const size_t row_bytes = (size_t)width * esz;
  const char* in = reinterpret_cast<const char*>(src);
  char* out = reinterpret_cast<char*>(dst);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return r;
  // dispatch: my sends read the send layout, my recvs land in the recv layout;
  // combine: the same messages reversed (send from the recv layout, land in the send layout)
  for (size_t i = 0; i < P.s_peer.size() && r == ncclSuccess; ++i) {
    const size_t bytes = (size_t)P.s_rows[i] * row_bytes;
    if (direction == 0)
      r = ncclSend(in + P.s_src[i] * row_bytes, bytes, ncclInt8, P.s_peer[i], comm, s);
    else
      r = ncclRecv(out + P.s_src[i] * row_bytes, bytes, ncclInt8, P.s_peer[i], comm, s);
  }
  for (size_t i = 0; i < P.r_peer.size() && r == ncclSuccess; ++i) {
    const size_t bytes = (size_t)P.r_rows[i] * row_bytes;
    if (direction == 0)
      r = ncclRecv(out + P.r_dst[i] * row_bytes, bytes, ncclInt8, P.r_peer[i], comm, s);
    else
      r = ncclSend(in + P.r_dst[i] * row_bytes, bytes, ncclInt8, P.r_peer[i], comm, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  return r != ncclSuccess ? r : r2;
}
#endif

}  // namespace moe
