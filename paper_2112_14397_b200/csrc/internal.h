// internal.h -- context, workspace carve-up and kernel launchers (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>

namespace moe { struct EpPlan; }
struct moe_ctx {
  int T, d, f, E, E_local, dtype, rank, world;
  void* comm;          // borrowed ncclComm_t (world > 1)
  int sm_count;
  int nblk;            // gate/dispatch token blocks = ceil(T / kGateBT)
  int dwg_splits;      // split-K factor for dW_g (SIMT path)
  int dwg_splits_max;  // capacity of `part` in splits (tcgen05 path)
  int use_tc;          // bf16 expert GEMMs on tcgen05 (1) or CUDA cores (0, MOE_GEMM=simt debug)
  // workspace (caller owned)
  uint8_t* ws;
  size_t ws_bytes;
  int* flags;          // [4] device error flags
  int* blk_cnt;        // [nblk, E]
  int* blk_base;       // [nblk, E]
  float* logits;       // [T, E] fp32 gate logits
  float* part;         // [dwg_splits, d, E] split-K partials of dW_g
  float* dxg;          // [T, d] fp32  dlogits W_g^T  (v1 path)
  float* colsum;       // [E] balance-loss column sums
  int* tot;            // [E] per-expert totals written by the dispatch scan
  float* colpart;      // [E_local, kColsumSplits, max(d, f)] bias-gradient partials
  int* rq;             // [1 + T] fp64-refine queue of the tcgen05 gate (count, tokens)
  int* tok_off;        // [2] = {0, roundup(T, 128)}: the token range as one row segment
  float* biasf;        // [E_local, roundup(f,256)] b1 then [E_local, roundup(d,256)] b2 in fp32 (tcgen05 epilogues)
  float* db2part;      // [E_local, db2_S, d] db2 column-sum partials (scratch within one call)
  int db2_S;           // row splits per expert of the fused combine_bwd
  // the (probs, slot) outputs of the most recent moe_dts_gate on this ctx: the per-block expert
  // counts it left in the workspace (blk_cnt) belong to them, and moe_dispatch / moe_ep2(d)_dispatch
  // refuse (MOE_EINVAL) any other pair -- the one piece of state carried from one call to the next
  const void* gate_probs;
  const void* gate_slot;
  unsigned long long gate_seq;
  void* gate_scratch;  // tcgen05 gate operands: W_g^T / [W_g|W_g] (bf16) and the hi|lo split of dL
  int* ep_counts;      // [world, E] gathered counts (EP)
  int* ep_off;         // [E_local + 1] recv-layout offsets (EP)
  int* ep_tot;         // [E_local] recv-layout rows per local expert (EP)
  int* ep2_scr;        // [E + 2] scan scratch of the fused peer-memory EP dispatch
  int* ep2_base;       // [E] first destination row of each global expert for this rank's tokens
  moe::EpPlan* ep;     // host exchange plan (EP), owned by the ctx
  int ep_G;            // GPUs per node for the hierarchical exchange (world = flat, the default)
  void* ep_stage;      // caller-owned relay staging rows of the hierarchical exchange
  long long ep_stage_rows;
};

namespace moe {
// NVLink peer pointers of one symmetric buffer, indexed by rank (fused peer-memory EP)
constexpr int kMaxPeers = 64;
struct PeerTable {
  const void* p[kMaxPeers];
};
struct EpPlan;
void ep_build_plan(EpPlan& P, const int* counts_all, int W, int E, int rank);
cudaError_t launch_zero_pads(const moe_ctx* c, void* buf, const int* offsets_dev, const int* tot_dev, int width,
                             cudaStream_t s);

constexpr int kGateBT = 128;   // tokens per gate/dispatch block

size_t workspace_bytes(const moe_ctx* c);
void carve_workspace(moe_ctx* c);

// ---------------------------------------------------------------- launchers
// All return cudaGetLastError() of the launch.
cudaError_t launch_spawn(const moe_ctx* c, const void* W1s, const void* b1s, const void* W2s,
                         const void* b2s, const uint32_t* M1, const uint32_t* M2, void* W1,
                         void* b1, void* W2, void* b2, cudaStream_t s);

cudaError_t launch_gate(const moe_ctx* c, const void* x, const void* Wg, const float* u, float tau,
                        float thr, int top1, float* probs, int32_t* slot, int32_t* counts,
                        int32_t* near_band, cudaStream_t s);

cudaError_t launch_dispatch(const moe_ctx* c, const void* x, const float* probs, int32_t* slot,
                            const int32_t* counts, void* x_perm, int32_t* row_token, float* row_gate,
                            int32_t* offsets, int64_t R_cap, int32_t* R_out, cudaStream_t s);

cudaError_t launch_combine(const moe_ctx* c, const void* e_out, const float* row_gate,
                           const int32_t* slot, void* y, cudaStream_t s);

cudaError_t launch_combine_bwd(moe_ctx* c, const void* dy, const void* e_out,
                               const float* row_gate, const int32_t* row_token,
                               const int32_t* offsets, int64_t R_cap, void* d_eout, float* dG_row,
                               float* db2, cudaStream_t s);

// db2[g] = column sums of the d_eout rows of local expert g (fixed-order partials + final)
cudaError_t launch_db2(moe_ctx* c, const void* d_eout, const int32_t* offsets, int64_t R_cap, float* db2,
                       cudaStream_t s);

// dx[t] (+)= sum_{e asc} dx_perm[slot[t,e]]   (accumulate: dx's current row starts the sum)
cudaError_t launch_dispatch_bwd(const moe_ctx* c, const void* dx_perm, const int32_t* slot, int accumulate,
                                void* dx, cudaStream_t s);

// counts: [count_rows][E] (1 = global counts, world = the all-gathered counts, summed per e);
// dx (optional): dx = dlogits W_g^T (the gate's input-gradient term, written)
cudaError_t launch_gate_bwd(const moe_ctx* c, const float* dG_row, const int32_t* slot,
                            const float* probs, const void* x, const void* Wg, float tau, float alpha,
                            const int32_t* counts, int count_rows, int64_t B_total, float* dWg, float* dlogits,
                            void* dx, cudaStream_t s);

cudaError_t launch_balance_loss(const moe_ctx* c, const float* probs, const int32_t* counts,
                                float alpha, int64_t B_total, float* loss, cudaStream_t s);

cudaError_t launch_expert_ffn(const moe_ctx* c, const void* x_perm, const int32_t* offsets,
                              int64_t R_cap, const void* W1, const void* b1, const void* W2,
                              const void* b2, void* gp, void* h, void* e_out, cudaStream_t s, const int32_t* arrive = nullptr,
                              const int32_t* arrive_target = nullptr);

cudaError_t launch_expert_ffn_bwd(moe_ctx* c, const void* d_eout, const void* x_perm,
                                  const void* gp, const void* h, const int32_t* offsets,
                                  int64_t R_cap, const void* W1, const void* W2, void* da,
                                  void* dx_perm, float* dW1, float* db1, float* dW2, float* db2,
                                  cudaStream_t s);

// ---------------------------------------------------------------- fused peer-memory EP ("ep2")
cudaError_t launch_ep2_counts(const moe_ctx* c, const int32_t* counts, const PeerTable& all, cudaStream_t s);
cudaError_t launch_ep2_plan(const moe_ctx* c, const int32_t* counts_all, int64_t R_cap, int32_t* offsets_recv,
                            cudaStream_t s);
cudaError_t launch_ep2_prepare(const moe_ctx* c, void* x_recv, int32_t* rtok, int32_t* rsrc, float* rgate,
                               int64_t R_cap, cudaStream_t s);
cudaError_t launch_ep2_dispatch(const moe_ctx* c, const void* x, const float* probs, int32_t* slot, const PeerTable& xr,
                                const PeerTable& rtok, const PeerTable& rsrc, const PeerTable& rgate, int64_t R_cap,
                                cudaStream_t s, const int32_t* sprefix = nullptr, int32_t* send = nullptr,
                                const PeerTable* arrive = nullptr);
cudaError_t launch_ep2_arrival_plan(const moe_ctx* c, const int32_t* counts_all, int32_t* sprefix, int32_t* target,
                                    cudaStream_t s);
cudaError_t launch_ep2_combine(const moe_ctx* c, const PeerTable& eo, const float* probs, const int32_t* slot, void* y,
                               cudaStream_t s);
bool ep2_width_ok(const moe_ctx* c);
cudaError_t launch_ep2_combine_bwd(moe_ctx* c, const PeerTable& dyp, const void* e_out, const float* rgate,
                                   const int32_t* rtok, const int32_t* rsrc, const int32_t* offsets, int64_t R_cap,
                                   void* d_eout, float* dG_row, float* db2, cudaStream_t s);
cudaError_t launch_ep2_dispatch_bwd(const moe_ctx* c, const PeerTable& dxp, const int32_t* slot, int accumulate,
                                    void* dx, cudaStream_t s, int slot_cols = 0, int cols_per_rank = 0);
// ep2 with token dedup (one row per (token, owner) each way)
cudaError_t launch_ep2d_dispatch(const moe_ctx* c, const void* x, const float* probs, int32_t* slot, int32_t* uslot,
                                 const PeerTable& tb, const PeerTable& urows, const PeerTable& rtok,
                                 const PeerTable& rsrc, const PeerTable& rgate, const PeerTable& ruid, int64_t R_cap,
                                 cudaStream_t s);
cudaError_t launch_ep2d_permute(const moe_ctx* c, const void* tokbuf, const int32_t* rtok, int32_t* ruid,
                                int64_t R_cap, void* x_recv, cudaStream_t s);
cudaError_t launch_ep2d_presum(const moe_ctx* c, const void* rows, const float* gate, const int32_t* urows, void* out,
                               cudaStream_t s);
cudaError_t launch_ep2d_gather_dy(const moe_ctx* c, const PeerTable& dyp, const int32_t* urows, void* dyu,
                                  cudaStream_t s);
cudaError_t launch_ep2d_combine(const moe_ctx* c, const PeerTable& ys, const int32_t* uslot, void* y, cudaStream_t s);
cudaError_t launch_ep2d_combine_bwd(moe_ctx* c, const void* dyu, const void* e_out, const float* rgate,
                                    const int32_t* ruid, const int32_t* offsets, int64_t R_cap, void* d_eout,
                                    float* dG_row, float* db2, cudaStream_t s);
cudaError_t launch_gate_bwd_peer(const moe_ctx* c, const PeerTable& dGp, const int32_t* slot, const float* probs,
                                 const void* x, const void* Wg, float tau, float alpha, const int32_t* counts,
                                 int count_rows, int64_t B_total, float* dWg, float* dlogits, void* dx,
                                 cudaStream_t s);

// ---------------------------------------------------------------- tcgen05 grouped GEMM (bf16)
bool tc_available();
cudaError_t tc_expert_ffn(const moe_ctx* c, const void* x_perm, const int32_t* offsets, int64_t R_cap,
                          const void* W1, const void* b1, const void* W2, const void* b2, void* gp, void* h,
                          void* e_out, cudaStream_t s, const int32_t* arrive = nullptr,
                          const int32_t* arrive_target = nullptr);
cudaError_t tc_expert_ffn_bwd(const moe_ctx* c, const void* d_eout, const void* x_perm, const void* gp,
                              const void* h, const int32_t* offsets, int64_t R_cap, const void* W1,
                              const void* W2, void* da, void* dx_perm, float* dW1, float* dW2, float* db1,
                              cudaStream_t s);
// db1[g][n] = sum over the 32-row blocks of group g of part[rb][n]  (fixed order)
cudaError_t launch_db1_reduce(const float* part, int N, const int* m_off, int G, float* out, float* part2,
                              long long R_cap, cudaStream_t s);

// ---------------------------------------------------------------- tcgen05 gate contractions (bf16)
bool gate_tc_supported(const moe_ctx* c);
cudaError_t gate_tc_forward(const moe_ctx* c, const void* x, const void* Wg, const float* u, float tau, float thr,
                            int top1, float* probs, int32_t* slot, int32_t* counts, int32_t* near_band,
                            cudaStream_t s);
// have_split: the [hi | lo] bf16 operand rows of these dlogits were just written to gate_dl2_buffer
// by the same moe_dts_gate_bwd call (else they are rebuilt from dlogits first)
cudaError_t gate_tc_dx(const moe_ctx* c, const float* dlogits, const void* Wg, void* dx_bf16, bool have_split,
                       cudaStream_t s);
void* gate_dl2_buffer(const moe_ctx* c);   // [T, Kp] bf16 hi|lo operand rows inside gate_scratch
cudaError_t gate_tc_dwg(const moe_ctx* c, const void* x, const float* dlogits, float* dWg, bool have_split,
                        cudaStream_t s);
cudaError_t tc_dense_store(const moe_ctx* c, const void* A, long long rows, int K, const void* B, int N, void* out,
                           const int* offsets_dev, cudaStream_t s);
cudaError_t launch_gate_softmax_tpt(const moe_ctx* c, const float* logits, const float* u, float tau, float thr,
                                    int top1, float* probs, int32_t* slot, int32_t* counts, int32_t* near_band,
                                    cudaStream_t s);
cudaError_t launch_reduce_splits(const float* part, int splits, long long n, float* out, cudaStream_t s);

// ---------------------------------------------------------------- SIMT grouped GEMM
enum SimtEpi { EPI_F32 = 0, EPI_T = 1, EPI_BIAS_T = 2, EPI_BIAS_GELU = 3, EPI_GELU_BWD = 4 };

struct SimtGemm {
  const void* A; long long sAm, sAk, gA;   // A(m,k) = A[m*sAm + k*sAk] (+ g*gA)
  const void* B; long long sBk, sBn, gB;   // B(k,n) = B[k*sBk + n*sBn] (+ g*gB)
  void* C; long long sCm, gC;              // C(m,n) = C[m*sCm + n]     (+ g*gC / split*gC)
  int M, N, K;
  const int* m_off;   // row-grouped: group of a 64-row tile found in m_off[0..G]; rows global
  const int* k_off;   // K-grouped: group g = blockIdx.z, K range [k_off[g], k_off[g+1])
  int G;
  int k_split;        // single problem split-K (C + z*gC), 1 = none
  int64_t m_tiles;    // grid.y upper bound for row-grouped problems
  const void* bias; long long gBias;        // bias[n] (+ g*gBias)
  const void* aux;    // GELU' input, same layout as C
  void* C2;           // second output (h) for EPI_BIAS_GELU, same layout as C
};

// ta/tb: element types of A and B (0 f32, 1 bf16); tout: type of C for EPI_T/BIAS/GELU epilogues.
// Mixed-type combinations always use the fp32-output epilogue.
cudaError_t launch_simt_gemm(const SimtGemm& g, int ta, int tb, int tout, int epi, cudaStream_t s);

// out[g][n] = sum over rows of group g of X[r][n]  (fp32 out, deterministic two-phase;
// `part` = workspace [G, kColsumSplits, N] fp32)
constexpr int kColsumSplits = 8;
cudaError_t launch_colsum_grouped(const void* X, int tin, int N, const int* m_off, int G, float* out,
                                  float* part, cudaStream_t s);
// out[g][n] = sum_s part[g][s][n]  (fixed order)
cudaError_t launch_colsum_final(const float* part, int N, int S, int G, float* out, cudaStream_t s);

}  // namespace moe

namespace moe {
// Count of kernels this library has launched (moe_kernel_launch_count): every launch
// site calls count_launch() right after its <<<>>> so the number is a direct tally.
void count_launch(int n = 1);
}  // namespace moe
