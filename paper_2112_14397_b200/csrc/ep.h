// ep.h -- expert-parallel exchange plan (host side) shared by ep.cu and the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "internal.h"
#ifdef MOE_HAVE_NCCL
#include <nccl.h>
#endif

namespace moe {

struct EpPlan {
  int W = 0, E = 0, El = 0, rank = 0;
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
#endif

}  // namespace moe
