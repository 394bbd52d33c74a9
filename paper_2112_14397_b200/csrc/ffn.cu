// ffn.cu -- step 5 (grouped expert FFN) and its backward B5: launch orchestration.
//
// bf16: tcgen05/TMEM/TMA grouped GEMM (gemm_tc.cu) when available; f32: CUDA-core
// FFMA grouped GEMM (gemm_simt.cu).  Every GEMM reads the device offsets[] directly:
// no host synchronisation on the routing result.
#include "common.cuh"
#include "internal.h"

namespace moe {

static SimtGemm base_rows(const int32_t* offsets, int G, int64_t R_cap) {
  SimtGemm g{};
  g.m_off = offsets;
  g.G = G;
  g.k_split = 1;
  g.m_tiles = (R_cap + 63) / 64;
  return g;
}

// overlap mode on the CUDA-core path: one warp waits for every local expert's rows before the
// GEMMs (the tcgen05 path waits per expert inside the GEMM's TMA producer instead)
__global__ void ep2_wait_all_kernel(const int* __restrict__ arrive, const int* __restrict__ target, int El,
                                    int* __restrict__ flags) {
  for (int g = threadIdx.x; g < El; g += blockDim.x) {
    const int tgt = target[g];
    for (int spins = 0;; ++spins) {
      int v;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(arrive + g) : "memory");
      if ((int)((unsigned)v - (unsigned)tgt) >= 0) break;
      if (*reinterpret_cast<volatile int*>(flags) & kFlagCapacity) break;
      if (spins > (1 << 22)) {
        atomicOr(flags, kFlagArrival);
        break;
      }
      __nanosleep(256);
    }
  }
}

cudaError_t launch_expert_ffn(const moe_ctx* c, const void* x_perm, const int32_t* offsets, int64_t R_cap,
                              const void* W1, const void* b1, const void* W2, const void* b2, void* gp, void* h,
                              void* e_out, cudaStream_t s, const int32_t* arrive, const int32_t* arrive_target) {
  const int d = c->d, f = c->f, El = c->E_local, dt = c->dtype;
  cudaError_t e;
  if (c->use_tc)
    return tc_expert_ffn(c, x_perm, offsets, R_cap, W1, b1, W2, b2, gp, h, e_out, s, arrive, arrive_target);
  if (arrive) {
    ep2_wait_all_kernel<<<1, 32, 0, s>>>(arrive, arrive_target, El, c->flags), count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // GEMM1: a = x_perm W1_e^T + b1_e, h = GELU(a)
  SimtGemm g1 = base_rows(offsets, El, R_cap);
  g1.A = x_perm; g1.sAm = d; g1.sAk = 1;
  g1.B = W1; g1.sBk = 1; g1.sBn = d; g1.gB = (long long)f * d;
  g1.C = gp; g1.sCm = f; g1.C2 = h;
  g1.bias = b1; g1.gBias = f;
  g1.M = 0; g1.N = f; g1.K = d;
  if ((e = launch_simt_gemm(g1, dt, dt, dt, EPI_BIAS_GELU, s)) != cudaSuccess) return e;
  if (!W2) return cudaSuccess;          // recompute call: GEMM1 only
  // GEMM2: e_out = h W2_e^T + b2_e
  SimtGemm g2 = base_rows(offsets, El, R_cap);
  g2.A = h; g2.sAm = f; g2.sAk = 1;
  g2.B = W2; g2.sBk = 1; g2.sBn = f; g2.gB = (long long)d * f;
  g2.C = e_out; g2.sCm = d;
  g2.bias = b2; g2.gBias = d;
  g2.N = d; g2.K = f;
  return launch_simt_gemm(g2, dt, dt, dt, EPI_BIAS_T, s);
}

cudaError_t launch_expert_ffn_bwd(moe_ctx* c, const void* d_eout, const void* x_perm, const void* gp,
                                  const void* h, const int32_t* offsets, int64_t R_cap, const void* W1,
                                  const void* W2, void* da, void* dx_perm, float* dW1, float* db1, float* dW2,
                                  float* db2, cudaStream_t s) {
  const int d = c->d, f = c->f, El = c->E_local, dt = c->dtype;
  cudaError_t e;
  if (c->use_tc) {
    if ((e = tc_expert_ffn_bwd(c, d_eout, x_perm, gp, h, offsets, R_cap, W1, W2, da, dx_perm, dW1, dW2, db1, s)) !=
        cudaSuccess)
      return e;
    return db2 ? launch_db2(c, d_eout, offsets, R_cap, db2, s) : cudaSuccess;
  }
  // dgrad2 + GELU': da = (d_eout W2_e) (.) GELU'(a)      (da may alias a)
  SimtGemm g = base_rows(offsets, El, R_cap);
  g.A = d_eout; g.sAm = d; g.sAk = 1;
  g.B = W2; g.sBk = f; g.sBn = 1; g.gB = (long long)d * f;
  g.C = da; g.sCm = f; g.aux = gp;
  g.N = f; g.K = d;
  if ((e = launch_simt_gemm(g, dt, dt, dt, EPI_GELU_BWD, s)) != cudaSuccess) return e;
  // wgrad2: dW2_e [d, f] = d_eout_e^T h_e   (ragged K = rows of e)
  SimtGemm w2{};
  w2.A = d_eout; w2.sAm = 1; w2.sAk = d;
  w2.B = h; w2.sBk = f; w2.sBn = 1;
  w2.C = dW2; w2.sCm = f; w2.gC = (long long)d * f;
  w2.M = d; w2.N = f; w2.K = 0; w2.k_off = offsets; w2.G = El; w2.k_split = 1;
  if ((e = launch_simt_gemm(w2, dt, dt, 0, EPI_F32, s)) != cudaSuccess) return e;
  // wgrad1: dW1_e [f, d] = da_e^T x_perm_e
  SimtGemm w1{};
  w1.A = da; w1.sAm = 1; w1.sAk = f;
  w1.B = x_perm; w1.sBk = d; w1.sBn = 1;
  w1.C = dW1; w1.sCm = d; w1.gC = (long long)f * d;
  w1.M = f; w1.N = d; w1.K = 0; w1.k_off = offsets; w1.G = El; w1.k_split = 1;
  if ((e = launch_simt_gemm(w1, dt, dt, 0, EPI_F32, s)) != cudaSuccess) return e;
  // dgrad1: dx_perm = da W1_e
  SimtGemm g1 = base_rows(offsets, El, R_cap);
  g1.A = da; g1.sAm = f; g1.sAk = 1;
  g1.B = W1; g1.sBk = d; g1.sBn = 1; g1.gB = (long long)f * d;
  g1.C = dx_perm; g1.sCm = d;
  g1.N = d; g1.K = f;
  if ((e = launch_simt_gemm(g1, dt, dt, dt, EPI_T, s)) != cudaSuccess) return e;
  // bias gradients: column sums per expert (pad rows are zero)
  if (db2 && (e = launch_db2(c, d_eout, offsets, R_cap, db2, s)) != cudaSuccess) return e;
  return launch_colsum_grouped(da, dt, f, offsets, El, db1, c->colpart, s);
}

}  // namespace moe
