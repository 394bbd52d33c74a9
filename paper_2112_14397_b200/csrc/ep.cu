// ep.cu -- expert parallelism (EP, GShard-style): experts split E/W per rank,
// tokens data-parallel.  The exchange plan is pure host arithmetic on the gathered
// per-(rank, expert) counts; the row exchanges are grouped ncclSend/ncclRecv over
// NVLink/NVSwitch, one message per (peer, local expert) segment, written straight into
// the receiver's expert-major, 128-row-aligned layout (no re-layout pass).
//
//   token side  ("send" layout): moe_dispatch's global-expert-major layout, offsets_send
//   expert side ("recv" layout): local expert j holds the rows of every source rank q in
//                                ascending q (= ascending global token index), 128-aligned
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
