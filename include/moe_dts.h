/*
 * moe_dts.h -- C ABI of the B200-native DTS-Gate MoE layer (EvoMoE, arXiv 2112.14397).
 *
 * One MoE FFN layer under the Dense-to-Sparse gate: forward and backward, plus the
 * expert-diversify spawn.  Citations are PAPER.md line numbers (P:n) with the
 * equation / algorithm they fall in; readings R1..R21 are listed in DESIGN.md.
 *
 * Conventions (all calls)
 *  - Every tensor pointer is a DEVICE pointer owned by the caller (allocated with
 *    torch or cudaMalloc).  The library never allocates or frees caller memory; the
 *    only memory it uses besides the caller's tensors is the caller-provided
 *    workspace (moe_set_workspace).
 *  - Layouts are row-major, element strides implied by the dims stored in the ctx.
 *    "D" is the activation/weight storage dtype chosen at moe_create (MOE_F32 or
 *    MOE_BF16); gate probabilities, combine weights and weight gradients are fp32.
 *  - Every compute call enqueues asynchronously on `stream` (a cudaStream_t, may be
 *    NULL for the legacy default stream) and returns a moe_status.  Host-side
 *    validation is synchronous: MOE_EINVAL for a bad scalar or a NULL required
 *    pointer, MOE_ESHAPE for bad dims.  moe_last_error() returns a thread-local
 *    message for the last failing call.  No C++ exception crosses the ABI.
 *  - Device-detected faults (non-finite gate logits -> MOE_ENONFINITE, row capacity
 *    exceeded -> MOE_ECAPACITY) set a flag in the workspace; they are returned by
 *    moe_check(), which synchronises `stream`.
 *  - No hidden state between calls, with ONE documented exception: moe_dts_gate leaves per-block
 *    expert counts in the workspace for the moe_dispatch / moe_ep2(d)_dispatch that consumes its
 *    (probs, slot); those calls return MOE_EINVAL for any other (probs, slot) pair (the ctx
 *    records the pointers of the most recent moe_dts_gate).  Every other value that flows from
 *    one call to the next is an explicit argument (db2 out of moe_combine_bwd, dx out of
 *    moe_dts_gate_bwd into an accumulating moe_dispatch_bwd).
 *  - Expert-major permuted ("row") layout: rows of expert e occupy
 *    [offsets[e], offsets[e] + counts[e]) in ascending token order (stable), followed
 *    by zero pad rows up to offsets[e+1]; offsets[e] is a multiple of 128
 *    (MOE_ROW_ALIGN).  R_pad = offsets[E].  Buffers in row layout have R_cap rows,
 *    R_cap >= R_pad (the caller sizes them, e.g. from counts copied to the host).
 */
#ifndef MOE_DTS_H
#define MOE_DTS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_ABI_VERSION 2
#define MOE_ROW_ALIGN 128

typedef enum {
  MOE_OK = 0,
  MOE_EINVAL = 1,      /* bad scalar argument (tau <= 0 or non-finite, c not in [0,1)), NULL pointer */
  MOE_ESHAPE = 2,      /* bad dims: E < 1, E % world != 0, d or d_ff not a multiple of 8 (bf16) / 4 (f32) */
  MOE_EDTYPE = 3,      /* unknown dtype */
  MOE_ECUDA = 4,       /* a CUDA runtime call failed (message has the CUDA error string) */
  MOE_ENCCL = 5,       /* an NCCL call failed */
  MOE_ENONFINITE = 6,  /* device: a gate logit was NaN/Inf ("NaN is an error state") */
  MOE_ECAPACITY = 7,   /* device: R_pad > R_cap; rows beyond R_cap were not written */
  MOE_EWORKSPACE = 8,  /* workspace missing or too small */
  MOE_EARRIVAL = 9     /* device: overlap mode, an expert's rows did not all arrive (bounded wait timed out) */
} moe_status;

typedef enum { MOE_F32 = 0, MOE_BF16 = 1 } moe_dtype;

typedef struct moe_ctx moe_ctx;

/* ---------------------------------------------------------------- lifecycle */

/* Create a layer context.  T = tokens on this rank, E = global number of experts,
 * world = expert-parallel group size (E_local = E / world experts live on `rank`).
 * nccl_comm: an ncclComm_t (borrowed, never destroyed) or NULL when world == 1.
 * d_model and d_ff: multiples of 8 (bf16; 16-byte rows) or 4 (f32).  bf16 layers whose d_model
 * and d_ff are both multiples of 64 run the tensor-core GEMMs and gate (64-wide K boxes); other
 * bf16 shapes run the CUDA-core GEMMs and the warp-per-token gate (same results, slower).
 * Returns MOE_ESHAPE / MOE_EDTYPE / MOE_EINVAL on bad arguments. */
int moe_create(moe_ctx** out, int T, int d_model, int d_ff, int E, int dtype,
               void* nccl_comm, int rank, int world);
int moe_destroy(moe_ctx* ctx);

/* Thread-local message describing the last error returned on this thread. */
const char* moe_last_error(void);
int moe_abi_version(void);

/* Process-wide count of CUDA kernels this library has launched (all contexts).  Used
 * by bench.py to report the number of library kernels inside the timed region. */
uint64_t moe_kernel_launch_count(void);

/* Workspace: device scratch owned by the caller, >= moe_workspace_bytes(ctx) bytes,
 * 256-byte aligned.  Holds per-block expert counts, the fp64-refine queue, split-K
 * partials and the device error flag. */
size_t moe_workspace_bytes(const moe_ctx* ctx);
int moe_set_workspace(moe_ctx* ctx, void* dev_ptr, size_t bytes);

/* Synchronise `stream`, read and clear the device error flag; returns MOE_OK,
 * MOE_ENONFINITE or MOE_ECAPACITY. */
int moe_check(moe_ctx* ctx, void* stream);

/* ---------------------------------------------------------------- forward */

/* Expert-diversify spawn (Alg. 1 lines 4-5; Fig. P:241-247).
 * For each LOCAL expert j (global id e = rank*E_local + j):
 *   W1[j] = W1s (.) M1_e,  W2[j] = W2s (.) M2_e,  b1[j] = b1s,  b2[j] = b2s  (R10).
 * W1s [d_ff, d], b1s [d_ff], W2s [d, d_ff], b2s [d]  (D, shared expert, nn.Linear [out,in]).
 * M1bits [E][ceil(d_ff*d/32)], M2bits [E][ceil(d*d_ff/32)] uint32 words, GLOBAL expert
 * index; bit (j % 32) of word j / 32 keeps flat element j (1 = keep).
 * Outputs W1 [E_local, d_ff, d], b1 [E_local, d_ff], W2 [E_local, d, d_ff], b2 [E_local, d].
 * One-time initialisation: there is no spawn backward (the paper defines none). */
int moe_dts_spawn(moe_ctx* ctx, const void* W1s, const void* b1s, const void* W2s, const void* b2s,
                  const uint32_t* M1bits, const uint32_t* M2bits,
                  void* W1, void* b1, void* W2, void* b2, void* stream);

/* DTS gate, steps 1-3 (Alg. 2; Eq. 6; Eq. 8; Eq. 9).
 *   L = x W_g;  zeta = -log(-log u);  p = softmax_E((L + zeta)/tau)        (R1, R2)
 *   dense (top1 == 0): m_i = [p_i > c] (strict, R3), argmax kept if none passes (R5)
 *   top1 (top1 != 0):  m = onehot(argmax p)   (Alg. 2 else-branch)
 *   G = p (.) m, NOT renormalised (R4).
 * x [T, d] D; Wg [d, E] D; u [T, E] fp32 in (0,1) or NULL (no noise).
 * Outputs: probs [T, E] fp32 (g'); slot [T, E] int32 (>= 0 selected, -1 not; the
 * row index is filled in by moe_dispatch); counts [E] int32 (this rank's tokens per
 * GLOBAL expert); near_band [1] int32 = #tokens with some |p - c| < 1e-6 (or, for
 * argmax-decided tokens, top-2 gap < 1e-6) -- the band reported by the tests (R18).
 * Entries within 5e-5 of the decision boundary are recomputed in fp64 before the
 * decision.  Errors: MOE_EINVAL if tau <= 0 or not
 * finite, c not in [0,1), or a required pointer is NULL. */
int moe_dts_gate(moe_ctx* ctx, const void* x, const void* Wg, const float* u, float tau,
                 float threshold, int top1, float* probs, int32_t* slot, int32_t* counts,
                 int32_t* near_band, void* stream);

/* Dispatch, step 4 (Alg. 1 lines 9-12 P:299-304; EP P:227).  Uses the per-block
 * counts left in the workspace by the preceding moe_dts_gate on the same stream; probs and
 * slot must be that call's outputs, unmodified (else MOE_EINVAL: "not the outputs of the most
 * recent moe_dts_gate").
 * Writes offsets [E+1] int32 (128-aligned exclusive prefix of counts), fills
 * slot[t,e] with the row index, row_token [R_cap] int32 (-1 on pad rows),
 * row_gate [R_cap] fp32 (= probs[t,e]; 0 on pads), x_perm [R_cap, d] D (copy of x_t;
 * 0 on pads) and R_out [1] int32 = offsets[E].  Rows >= R_cap are not written and
 * raise MOE_ECAPACITY at the next moe_check. */
int moe_dispatch(moe_ctx* ctx, const void* x, const float* probs, int32_t* slot,
                 void* x_perm, int32_t* row_token, float* row_gate, int32_t* offsets,
                 int64_t R_cap, int32_t* R_out, void* stream);

/* Grouped expert FFN, step 5 (Eq. 3 P:169-172 with GELU erf form P:472, R8).
 * For every row r of expert e (rows [offsets[e], offsets[e+1])):
 *   a = W1[e] x_perm[r] + b1[e];  h[r] = GELU(a) = a Phi(a);  e_out[r] = W2[e] h[r] + b2[e]
 * and, for the backward, gp[r] = GELU'(a) = Phi(a) + a phi(a), computed in the same
 * epilogue from the same Phi(a) and exp(-a^2/2) (the pre-activation a itself is not kept).
 * gp_saved, h_saved [R_cap, d_ff] D; e_out [R_cap, d] D.  W1..b2 are LOCAL experts
 * (moe_dts_spawn layout).  bf16: tcgen05 tensor cores, fp32 accumulation; f32: fp32
 * CUDA-core FMA. */
int moe_expert_ffn(moe_ctx* ctx, const void* x_perm, const int32_t* offsets, int64_t R_cap,
                   const void* W1, const void* b1, const void* W2, const void* b2,
                   void* gp_saved, void* h_saved, void* e_out, void* stream);

/* NEXT #3, MoE-aware recomputation.  moe_expert_ffn may be called with
 * gp_saved == NULL: GEMM1's epilogue then writes only h (a transient buffer the caller may
 * reuse after the call), and nothing [R, d_ff]-sized is kept until the backward.  Before
 * moe_expert_ffn_bwd, moe_expert_ffn_recompute re-runs GEMM1 + GELU from the kept x_perm
 * (the expert-side input, which under EP is the received all-to-all buffer: no exchange is
 * repeated) and writes gp_saved and h_saved.  Costs one extra GEMM1 (1/6 of the FLOPs). */
int moe_expert_ffn_recompute(moe_ctx* ctx, const void* x_perm, const int32_t* offsets, int64_t R_cap,
                             const void* W1, const void* b1, void* gp_saved, void* h_saved, void* stream);

/* Combine + un-permute, step 6 (Eq. 4, Eq. 7, Alg. 1 line 11):
 *   y[t] = sum over selected e in ASCENDING e of row_gate[slot[t,e]] * e_out[slot[t,e]]
 * accumulated in fp32 (R14), stored as D.  y [T, d]. */
int moe_combine(moe_ctx* ctx, const void* e_out, const float* row_gate, const int32_t* slot,
                void* y, void* stream);

/* ---------------------------------------------------------------- backward */

/* Combine backward (chain rule of Eq. 7).  For every row r < offsets[E]:
 *   t = row_token[r];  d_eout[r] = row_gate[r] * dy[t];  dG_row[r] = <dy[t], e_out[r]>
 * (0 for pad rows).  dy [T, d] D; d_eout [R_cap, d] D; dG_row [R_cap] fp32.
 * db2 [E, d] fp32 (optional, NULL = not computed): the per-expert column sums of the d_eout
 * rows this call stores (= the expert FFN's b2 gradient, chain rule of Eq. 3), fused into the
 * same pass; pass db2 = NULL to moe_expert_ffn_bwd then.  Single-rank ctx only (MOE_EINVAL
 * under the NCCL exchange, where db2 is an expert-side sum over the received rows). */
int moe_combine_bwd(moe_ctx* ctx, const void* dy, const void* e_out, const float* row_gate,
                    const int32_t* row_token, const int32_t* offsets, int64_t R_cap,
                    void* d_eout, float* dG_row, float* db2, void* stream);

/* Expert FFN backward (chain rule of Eq. 3).  Per expert e over its rows:
 *   dh = d_eout W2[e];  da = dh (.) gp   (gp = GELU'(a) saved by moe_expert_ffn)
 *   dW2[e] = d_eout^T h;  db2[e] = colsum(d_eout);  dW1[e] = da^T x_perm;  db1[e] = colsum(da)
 *   dx_perm = da W1[e]
 * da [R_cap, d_ff] D may ALIAS gp_saved (overwritten in place).  dW1 [E_local, d_ff, d],
 * db1 [E_local, d_ff], dW2 [E_local, d, d_ff], db2 [E_local, d] fp32 (overwritten).  db2 may be
 * NULL (it was taken from moe_combine_bwd); otherwise it is summed from the d_eout given here,
 * with the same partition and order as moe_combine_bwd's (bit-identical). */
int moe_expert_ffn_bwd(moe_ctx* ctx, const void* d_eout, const void* x_perm, const void* gp_saved,
                       const void* h_saved, const int32_t* offsets, int64_t R_cap,
                       const void* W1, const void* W2, void* da, void* dx_perm,
                       float* dW1, float* db1, float* dW2, float* db2, void* stream);

/* Gate backward (softmax Jacobian; mask, u and tau are constants).  Per token:
 *   dp_e = m_e dG[slot[t,e]] (+ balance term alpha N count_e / B^2 if balance_alpha > 0,
 *          Eq. 10, counts = global counts, B = global batch size)
 *   dz = p (.) (dp - <p, dp>);  dlogits = dz / tau;   dWg = x^T dlogits  (fp32, [d, E])
 *   dx = dlogits W_g^T  (D, [T, d]; written when dx != NULL, Wg [d, E] then required)
 * dlogits [T, E] fp32 is an output.  counts may be NULL when balance_alpha == 0.  The expert
 * path's input gradient is then added onto dx by moe_dispatch_bwd(accumulate = 1). */
int moe_dts_gate_bwd(moe_ctx* ctx, const float* dG_row, const int32_t* slot, const float* probs,
                     const void* x, const void* Wg, float tau, float balance_alpha, const int32_t* counts,
                     int64_t B_total, float* dWg, float* dlogits, void* dx, void* stream);

/* Dispatch backward (inverse of step 4):
 *   dx[t] = (accumulate ? dx[t] : 0) + sum over selected e in ASCENDING e of dx_perm[slot[t,e]]
 * accumulated in fp32 from the stored dx row, stored as D.  With accumulate = 1 after
 * moe_dts_gate_bwd(dx) this is the layer's full input gradient. */
int moe_dispatch_bwd(moe_ctx* ctx, const void* dx_perm, const int32_t* slot, int accumulate, void* dx,
                     void* stream);

/* ---------------------------------------------------------------- expert parallelism */
/* EP (GShard-style): E/world experts per rank (global ids rank*E_local ...),
 * tokens data-parallel.  Per layer pass: moe_dts_gate -> moe_ep_exchange_counts ->
 * moe_ep_plan -> moe_ep_upload -> moe_dispatch (token side, "send" layout over all E
 * experts) -> moe_ep_dispatch (send -> expert side "recv" layout) -> moe_expert_ffn on the
 * recv layout -> moe_ep_combine (recv -> send) -> moe_combine.  Backward mirrors it:
 * combine_bwd(db2 = NULL) -> moe_ep_dispatch(d_eout) -> expert_ffn_bwd(db2) -> moe_ep_combine(dx_perm)
 * -> gate_bwd(dx) -> moe_ep_allreduce(dWg) -> dispatch_bwd(accumulate = 1).
 * Recv layout: local expert j occupies [offsets_recv[j], offsets_recv[j+1]) (128-aligned);
 * inside it the rows of source rank 0, 1, ... in order (ascending global token index);
 * pad rows are zeroed by moe_ep_dispatch.  Messages: one ncclSend/ncclRecv per
 * (peer, local expert) segment inside one NCCL group, written in place (no re-layout). */

/* NCCL bootstrap helpers (the id is broadcast by the caller, e.g. with torch.distributed). */
int moe_nccl_unique_id(void* id_out, size_t bytes);   /* bytes >= 128 */
int moe_nccl_comm_init(void** comm_out, const void* id, int world, int rank);
int moe_nccl_comm_destroy(void* comm);

/* All-gather this rank's counts [E] (device) into counts_all_host [world][E] (host);
 * synchronises `stream` (the plan needs the counts on the host). */
int moe_ep_exchange_counts(moe_ctx* ctx, const int32_t* counts, int32_t* counts_all_host, void* stream);

/* Host-only: build the exchange plan from counts_all [world][E] (host) and return the
 * token-side offsets_send [E+1], expert-side offsets_recv [E_local+1] (either may be
 * NULL) and the row totals R_send, R_recv.  Needs no GPU.  MOE_EINVAL on counts < 0 or > T. */
int moe_ep_plan(moe_ctx* ctx, const int32_t* counts_all, int32_t* offsets_send, int32_t* offsets_recv,
                int64_t* R_send, int64_t* R_recv);

/* Host-only accessor for tests: which = 0 -> this rank's sends (peer, send-layout row, rows),
 * which = 1 -> its receives (peer, recv-layout row, rows), in NCCL posting order. */
int moe_ep_plan_chunks(moe_ctx* ctx, int which, int32_t* peer, int64_t* row, int32_t* nrows, int max_chunks,
                       int* n_out);

/* Copy the plan's offsets_recv to a device buffer (and the library's pad table); syncs. */
int moe_ep_upload(moe_ctx* ctx, int32_t* offsets_recv_dev, void* stream);

/* Row exchange of `width`-element D rows: send layout -> recv layout (zeroing recv pads),
 * and the reverse.  MOE_ECAPACITY if R_recv_cap < the plan's R_recv; MOE_ENCCL on NCCL errors. */
int moe_ep_dispatch(moe_ctx* ctx, const void* send_rows, void* recv_rows, int width, int64_t R_recv_cap,
                    void* stream);
int moe_ep_combine(moe_ctx* ctx, const void* recv_rows, void* send_rows, int width, void* stream);

/* ---- NEXT #4: topology-aware hierarchical all-to-all ----
 * For multi-node EP (nodes of gpus_per_node consecutive ranks).  Rows from node A to node
 * B != A go source -> relay(A,B) (intra-node gather; relay(X,Y) = local GPU Y mod G of node X)
 * -> relay(B,A) (ONE inter-node message per ordered node pair, aggregating the G^2 GPU-pair
 * payloads: the paper's "#GPU^2 times larger" message) -> destination (intra-node scatter,
 * written straight into the recv layout).  Same-node rows go directly.  The recv / send
 * layouts and the results are identical to the flat exchange; only the message set differs.
 * moe_ep_set_topology: gpus_per_node must divide world; world (the default) = flat.  Call
 * before moe_ep_plan.  After the plan, moe_ep_stage_rows gives the relay staging rows this
 * rank needs; the caller owns a buffer of that many `width`-element D rows and passes it
 * with moe_ep_set_stage before moe_ep_dispatch / moe_ep_combine (MOE_ECAPACITY otherwise). */
int moe_ep_set_topology(moe_ctx* ctx, int gpus_per_node);
int moe_ep_stage_rows(moe_ctx* ctx, int64_t* rows);
int moe_ep_set_stage(moe_ctx* ctx, void* stage, int64_t rows_cap);
/* Host-only accessor for tests: the messages of hierarchical phase 0 / 1 / 2 (dispatch
 * direction), sends (is_recv = 0) or receives, in NCCL posting order: peer, buffer
 * (0 send layout, 1 recv layout, 2 relay gather stage, 3 relay receive stage; stage 3 starts
 * after the gather stage's rows), row offset and rows.  n_out = 0 for a flat plan. */
int moe_ep_hier_chunks(moe_ctx* ctx, int phase, int is_recv, int32_t* peer, int32_t* buf, int64_t* row,
                       int32_t* nrows, int max_chunks, int* n_out);
/* Host-only cost-model identities of both plans on a virtual topology (no ctx, no GPU) for
 * routing counts_all [world][E]: stats[8] = { flat inter-node (src, dst) GPU pairs with
 * payload, flat inter-node rows, flat intra-node rows, hierarchical inter-node messages,
 * hierarchical inter-node rows, hierarchical intra-node rows moved, ordered node pairs with
 * payload, largest inter-node message (rows) }. */
int moe_ep_topology_stats(int world, int gpus_per_node, int E, const int32_t* counts_all, int64_t* stats);

/* In-place sum all-reduce over the EP group: fp32 (dW_g, C6) or int32 (global counts, C7). */
int moe_ep_allreduce(moe_ctx* ctx, void* buf, int64_t n, int is_int32, void* stream);

/* ---------------------------------------------------------------- fused peer-memory EP ("ep2")
 * The B200-native expert-parallel path: the all-to-all exchanges are fused into the routing
 * kernels as NVLink peer loads / stores (P:226-227 data flow, no NCCL send/recv of rows).
 * Every rank's row buffers are symmetric (mapped into every rank, e.g. torch symmetric
 * memory / CUDA IPC); the `*_peers` arguments are HOST arrays of `world` device pointers
 * (entry q = that buffer on rank q, entry rank = the local one).  Per step:
 *   moe_dts_gate -> moe_ep2_counts (counts row into every rank's counts_all) -> barrier ->
 *   moe_ep2_plan (device: recv offsets, destination bases) -> moe_ep2_prepare_recv (pad rows)
 *   -> moe_ep2_dispatch (scan + rank: slot[t,e] = row on rank e/E_local, row metadata stored at
 *   the owner; copy: x rows stored into the owners' x_recv) -> barrier -> moe_expert_ffn on
 *   x_recv -> barrier -> moe_ep2_combine (token side gathers e_out rows from the owners).
 *   Backward: barrier -> moe_ep2_combine_bwd (expert side reads dy rows from the token
 *   owners; d_eout, dG_row and db2 locally) -> moe_expert_ffn_bwd(db2 = NULL) -> barrier ->
 *   moe_ep2_gate_bwd (dG from the owners; dx = dlogits W_g^T) -> moe_ep_allreduce(dWg) ->
 *   moe_ep2_dispatch_bwd(accumulate = 1) (dx_perm rows from the owners).
 * moe_ep2_gate_bwd's balance term takes counts_all [world][E] (this rank's copy, filled by
 * moe_ep2_counts): the kernel sums the rows, i.e. uses the GLOBAL counts of Eq. 10.
 * Layouts (recv layout of each rank, expert-major, sources in rank order) and results equal
 * the NCCL path's and, for the global token set, the single-rank layer's.  No host sync:
 * R_recv_cap is a static capacity, a multiple of 128 (worst case world*T*E_local + 127*E_local,
 * rounded up); overflow raises
 * MOE_ECAPACITY at moe_check.  moe_ep2(d)_combine_bwd fuses the db2 partials into its row pass
 * up to d_model = 1024 (bf16) / 512 (f32); wider rows take a warp-per-row pass plus a db2 pass.
 * nccl_comm == MOE_COMM_EMULATED (moe_create) runs `world` ranks in ONE process on one device
 * (the tests): moe_ep2_barrier is then a no-op and the caller orders the ranks' launches;
 * the NCCL exchange calls refuse such a ctx. */
#define MOE_COMM_EMULATED ((void*)1)
int moe_ep2_barrier(moe_ctx* ctx, void* stream);
int moe_ep2_counts(moe_ctx* ctx, const int32_t* counts, int32_t* const* counts_all_peers, void* stream);
int moe_ep2_plan(moe_ctx* ctx, const int32_t* counts_all, int64_t R_recv_cap, int32_t* offsets_recv, void* stream);
int moe_ep2_prepare_recv(moe_ctx* ctx, void* x_recv, int32_t* rtok, int32_t* rsrc, float* rgate,
                         int64_t R_recv_cap, void* stream);
int moe_ep2_dispatch(moe_ctx* ctx, const void* x, const float* probs, int32_t* slot, void* const* x_recv_peers,
                     int32_t* const* rtok_peers, int32_t* const* rsrc_peers, float* const* rgate_peers,
                     int64_t R_recv_cap, void* stream);
/* Exchange / GEMM overlap ("low utilization of network bandwidth"): the x
 * exchange and the expert GEMMs without a barrier between them.  Sequence per rank:
 *   moe_ep2_counts -> barrier -> moe_ep2_plan -> moe_ep2_arrival_plan -> moe_ep2_prepare_recv ->
 *   moe_ep2_dispatch_ordered -> moe_ep2_expert_ffn (no barrier) -> barrier -> moe_ep2_combine.
 * moe_ep2_arrival_plan: sprefix [E+1] int32 (device, caller-owned) = prefix of THIS rank's counts
 *   (row `rank` of counts_all) in (local expert j, owner p) order, index j*world + p; arrive_target
 *   [E_local] int32 (device, caller-owned, zero before the first step, never reset) += the rows all
 *   sources send to each of this rank's local experts this step (uint32 wrap-around arithmetic).
 * moe_ep2_dispatch_ordered: as moe_ep2_dispatch, plus the send list send [T*E] int32 (device scratch,
 *   caller-owned, any contents; entry i = the token of the i-th (token, expert) pair in sprefix
 *   order) and arrive_peers (world device pointers to every rank's [E_local] int32 arrival counters,
 *   symmetric memory, zero before the first step, never reset): the copy pass walks the send list
 *   in order, so every owner's local expert 0 is filled first, and after each chunk of 256 entries
 *   adds the chunk's per-(owner, expert) entry counts to the owner's counters with a system-scope
 *   release (dropped rows of an overflowing step count too).
 * moe_ep2_expert_ffn: moe_expert_ffn on the recv layout whose GEMM1 TMA producer acquire-polls
 *   arrive[g] (this rank's counters) up to arrive_target[g] before an expert's first tile (the
 *   CUDA-core path: one wait for all experts before its GEMMs).  The wait ends early when the plan
 *   raised MOE_ECAPACITY and after a bounded spin raises MOE_EARRIVAL (at moe_check) instead of
 *   hanging.  Results are those of moe_ep2_dispatch + barrier + moe_expert_ffn, bit for bit. */
int moe_ep2_arrival_plan(moe_ctx* ctx, const int32_t* counts_all, int32_t* sprefix, int32_t* arrive_target,
                         void* stream);
int moe_ep2_dispatch_ordered(moe_ctx* ctx, const void* x, const float* probs, int32_t* slot, void* const* x_recv_peers,
                             int32_t* const* rtok_peers, int32_t* const* rsrc_peers, float* const* rgate_peers,
                             int64_t R_recv_cap, const int32_t* sprefix, int32_t* send, int32_t* const* arrive_peers,
                             void* stream);
int moe_ep2_expert_ffn(moe_ctx* ctx, const void* x_recv, const int32_t* offsets_recv, int64_t R_recv_cap,
                       const void* W1, const void* b1, const void* W2, const void* b2, void* gp_saved, void* h_saved,
                       void* e_out, const int32_t* arrive, const int32_t* arrive_target, void* stream);
int moe_ep2_combine(moe_ctx* ctx, void* const* e_out_peers, const float* probs, const int32_t* slot, void* y,
                    void* stream);
int moe_ep2_combine_bwd(moe_ctx* ctx, void* const* dy_peers, const void* e_out, const float* rgate,
                        const int32_t* rtok, const int32_t* rsrc, const int32_t* offsets_recv, int64_t R_recv_cap,
                        void* d_eout, float* dG_row, float* db2, void* stream);
int moe_ep2_gate_bwd(moe_ctx* ctx, float* const* dG_peers, const int32_t* slot, const float* probs, const void* x,
                     const void* Wg, float tau, float balance_alpha, const int32_t* counts_all, int64_t B_total,
                     float* dWg, float* dlogits, void* dx, void* stream);
int moe_ep2_dispatch_bwd(moe_ctx* ctx, void* const* dx_perm_peers, const int32_t* slot, int accumulate, void* dx,
                         void* stream);

/* ---------------------------------------------------------------- ep2 with token dedup ("ep2d")
 * SURVEY §8(e) "Dedup": a token is sent ONCE to every GPU owning any of its selected
 * experts, and each owner pre-sums its local experts' contributions before the return trip,
 * so the NVLink bytes per (token, owner) are one row each way instead of one per selected
 * expert (up to E_local x fewer).  Unique slot of token t of source rank s on every owner:
 * u = s * T + t.  Extra symmetric buffers per rank (U = world * T):
 *   tokbuf [U, d] (D), urows [U, E_local] int32 (expert-side row of (u, local expert j) or
 *   -1; rewritten whole every step by the token side), ruid [R_recv_cap] int32 (row -> u),
 *   ysum / dyu / dxu [U, d] (D); token side: uslot [T, world] int32 (u on owner q or -1).
 * Forward: gate -> ep2_counts -> barrier -> ep2_plan -> ep2_prepare_recv -> moe_ep2d_dispatch
 *   (rows, row metadata and ruid / urows at the owners, x stored once per owner into tokbuf)
 *   -> barrier -> moe_ep2d_permute (expert side, local: x_recv[r] = tokbuf[ruid[r]]) ->
 *   moe_expert_ffn -> moe_ep2d_presum(e_out, rgate) -> ysum (ysum[u] = sum_{j asc} G e_out,
 *   rounded to D) -> barrier -> moe_ep2d_combine (token side: y = sum_{q asc} ysum@q[uslot]).
 * Backward: dy staged in a symmetric buffer -> barrier -> moe_ep2d_gather_dy (expert side:
 *   dyu[u] = dy@s[t], one read per (token, owner)) -> moe_ep2d_combine_bwd (d_eout, dG, db2
 *   from dyu) -> moe_expert_ffn_bwd(db2 = NULL) -> moe_ep2d_presum(dx_perm, NULL) -> dxu ->
 *   barrier -> moe_ep2_gate_bwd(dx = dL W_g^T) -> moe_ep_allreduce(dWg) ->
 *   moe_ep2d_dispatch_bwd(accumulate = 1) (token side: dx += sum_{q asc} dxu@q[uslot]).
 * Routing, d_eout, dG, dlogits and the expert weight gradients equal the non-dedup path's bit
 * for bit; y and dx differ by the rounding of the per-owner partial sums to D (one extra
 * rounding per owner, ~2^-9 relative for bf16). */
int moe_ep2d_dispatch(moe_ctx* ctx, const void* x, const float* probs, int32_t* slot, int32_t* uslot,
                      void* const* tokbuf_peers, int32_t* const* urows_peers, int32_t* const* rtok_peers,
                      int32_t* const* rsrc_peers, float* const* rgate_peers, int32_t* const* ruid_peers,
                      int64_t R_recv_cap, void* stream);
/* also sets ruid = -1 on the pad rows of the recv layout (moe_ep2d_combine_bwd reads ruid) */
int moe_ep2d_permute(moe_ctx* ctx, const void* tokbuf, const int32_t* rtok, int32_t* ruid, int64_t R_recv_cap,
                     void* x_recv, void* stream);
/* out[u] = sum_{j asc, urows[u][j] >= 0} (rgate[row] *) rows[row]; rgate NULL = unweighted.
 * Unique slots with no row are left untouched. */
int moe_ep2d_presum(moe_ctx* ctx, const void* rows, const float* rgate_or_null, const int32_t* urows, void* out,
                    void* stream);
int moe_ep2d_gather_dy(moe_ctx* ctx, void* const* dy_peers, const int32_t* urows, void* dyu, void* stream);
int moe_ep2d_combine(moe_ctx* ctx, void* const* ysum_peers, const int32_t* uslot, void* y, void* stream);
int moe_ep2d_combine_bwd(moe_ctx* ctx, const void* dyu, const void* e_out, const float* rgate, const int32_t* ruid,
                         const int32_t* offsets_recv, int64_t R_recv_cap, void* d_eout, float* dG_row, float* db2,
                         void* stream);
int moe_ep2d_dispatch_bwd(moe_ctx* ctx, void* const* dxu_peers, const int32_t* uslot, int accumulate, void* dx,
                          void* stream);

/* ---------------------------------------------------------------- NEXT #1 */

/* Balance loss, Eq. 10: loss = alpha N sum_i (counts_i / B^2) sum_s p[s,i]
 * over this rank's probs (the caller all-reduces across ranks).  loss [1] fp32. */
int moe_balance_loss(moe_ctx* ctx, const float* probs, const int32_t* counts, float alpha,
                     int64_t B_total, float* loss, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_DTS_H */
