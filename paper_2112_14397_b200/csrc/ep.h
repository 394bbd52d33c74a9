// ep.h -- expert-parallel exchange plan (host side) shared by ep.cu and the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "internal.h"
#ifdef MOE_HAVE_NCCL
#include <nccl.h>
#endif

namespace moe {

// Topology-aware hierarchical exchange (NEXT #4): one message kind per phase.
// buf: 0 = token-side send layout, 1 = expert-side recv layout, 2 = relay gather stage
// (stage_out), 3 = relay receive stage (stage_in); row = row offset into that buffer.
struct EpMsg {
  int peer, buf;
  long long row;
  int rows;
};
struct EpHier {
  int G = 0, N = 0;                       // GPUs per node, nodes
  // dispatch-direction phases: 0 = intra-node (direct + gather to the relays),
  // 1 = inter-node relay <-> relay (one message per ordered node pair), 2 = intra-node scatter
  std::vector<EpMsg> snd[3], rcv[3];
  long long stage_out = 0, stage_in = 0;  // rows
};
// relay of node X for the traffic to / from node Y: local GPU (Y mod G) of node X
inline int ep_relay(int X, int Y, int G) { return X * G + (Y % G); }
void ep_build_hier(EpHier& H, const int* counts_all, int W, int E, int rank, int G,
                   const std::vector<int>& offsets_send_me);

struct EpPlan {
  int W = 0, E = 0, El = 0, rank = 0;
  int G = 0;                       // GPUs per node (hierarchical when W / G > 1)
  EpHier H;
  std::vector<int> offsets_send;   // [E+1]
  std::vector<int> offsets_recv;   // [El+1]
  std::vector<int> recv_tot;       // [El]
  // dispatch direction (token side -> expert side)
  std::vector<int> s_peer, s_rows;
  std::vector<long long> s_src;    // send-layout row
  std::vector<int> r_peer, r_rows;
  std::vector<long long> r_dst;    // recv-layout row
  long long R_send = 0, R_recv = 0;
};

#ifdef MOE_HAVE_NCCL
ncclResult_t ep_exchange(const moe_ctx* c, const EpPlan& P, const void* src, void* dst, int width, int direction,
                         cudaStream_t s);
// three NCCL groups (phases 0,1,2 for dispatch; 2,1,0 reversed for combine) through `stage`
// (stage_out rows, then stage_in rows, `width` elements each)
ncclResult_t ep_exchange_hier(const moe_ctx* c, const EpPlan& P, const void* src, void* dst, void* stage, int width,
                              int direction, cudaStream_t s);
#endif

}  // namespace moe
