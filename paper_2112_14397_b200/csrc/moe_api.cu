// moe_api.cu -- the extern "C" boundary (include/moe_dts.h): validation, workspace,
// error reporting.  Every compute call forwards to a kernel launcher in namespace moe.
#include <math.h>
#include <stdlib.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <new>
#include <string>

#include "../../include/moe_dts.h"
#include "common.cuh"
#include "internal.h"
#include "ep.h"

namespace {
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return MOE_OK;
  return fail(MOE_ECUDA, "%s: CUDA error %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define REQUIRE(p)                                                              \
  do {                                                                          \
    if ((p) == nullptr) return fail(MOE_EINVAL, "%s: argument '%s' is NULL", __func__, #p); \
  } while (0)

// token-sized arrays may be NULL when the rank holds no tokens (T == 0)
#define REQUIRE_T(p)                                                            \
  do {                                                                          \
    if ((p) == nullptr && ctx->T > 0)                                           \
      return fail(MOE_EINVAL, "%s: argument '%s' is NULL", __func__, #p);      \
  } while (0)
// row-sized arrays may be NULL when R_cap == 0
#define REQUIRE_R(p)                                                            \
  do {                                                                          \
    if ((p) == nullptr && R_cap > 0)                                            \
      return fail(MOE_EINVAL, "%s: argument '%s' is NULL", __func__, #p);      \
  } while (0)

int check_ctx(const moe_ctx* c, const char* fn) {
  if (!c) return fail(MOE_EINVAL, "%s: ctx is NULL", fn);
  if (!c->ws) return fail(MOE_EWORKSPACE, "%s: no workspace set (moe_set_workspace)", fn);
  return MOE_OK;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
}  // namespace

namespace moe {

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Carve {
  size_t flags, blk_cnt, blk_base, logits, part, dxg, colsum, tot, colpart, ep_counts, ep_off, ep_tot, gate_scratch, rq, tok_off, biasf, db2part, ep2_scr, ep2_base, total;
};

// row splits per expert for the fused combine_bwd + db2 partials: one wave of its 2 resident
// blocks per SM in total
static int db2_splits(const moe_ctx* c) {
  const int El = c->E_local > 0 ? c->E_local : 1;
  int S = 2 * (c->sm_count > 0 ? c->sm_count : 148) / El;
  return S < 1 ? 1 : (S > 128 ? 128 : S);
}

static Carve carve(const moe_ctx* c) {
  Carve k;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  k.flags = take(16 * sizeof(int));
  k.blk_cnt = take(sizeof(int) * (size_t)c->nblk * c->E);
  k.blk_base = take(sizeof(int) * (size_t)c->nblk * c->E);
  k.logits = take(sizeof(float) * (size_t)c->T * c->E);
  k.part = take(sizeof(float) * (size_t)(c->dwg_splits > c->dwg_splits_max ? c->dwg_splits : c->dwg_splits_max) *
                c->d * c->E);
  k.dxg = take(sizeof(float) * (size_t)c->T * c->d);
  k.colsum = take(sizeof(float) * (size_t)c->E);
  k.tot = take(sizeof(int) * (size_t)c->E);
  k.colpart = take(sizeof(float) * (size_t)c->E_local * kColsumSplits * (size_t)(c->d > c->f ? c->d : c->f));
  k.ep_counts = take(sizeof(int) * (size_t)c->world * c->E);
  k.ep_off = take(sizeof(int) * (size_t)(c->E_local + 1));
  k.ep_tot = take(sizeof(int) * (size_t)c->E_local);
  {
    const size_t Ep = (c->E + 15) / 16 * 16, Kp = (2 * Ep + 63) / 64 * 64;
    const size_t a = Ep * c->d, b = Kp * (c->d + (size_t)c->T);
    k.gate_scratch = take(2 * (a > b ? a : b));
  }
  k.rq = take(sizeof(int) * ((size_t)c->T + 1));
  k.tok_off = take(sizeof(int) * 2);
  // fp32 copies of b1 / b2 for the tensor-core epilogues, rows padded to 256 columns
  k.biasf = take(sizeof(float) * (size_t)c->E_local * (size_t)((c->f + 255) / 256 * 256 + (c->d + 255) / 256 * 256));
  k.db2part = take(sizeof(float) * (size_t)c->E_local * (size_t)db2_splits(c) * (size_t)c->d);
  k.ep2_scr = take(sizeof(int) * ((size_t)c->E + 2));
  k.ep2_base = take(sizeof(int) * (size_t)c->E);
  k.total = o;
  return k;
}

size_t workspace_bytes(const moe_ctx* c) { return carve(c).total; }

void carve_workspace(moe_ctx* c) {
  Carve k = carve(c);
  c->flags = reinterpret_cast<int*>(c->ws + k.flags);
  c->blk_cnt = reinterpret_cast<int*>(c->ws + k.blk_cnt);
  c->blk_base = reinterpret_cast<int*>(c->ws + k.blk_base);
  c->logits = reinterpret_cast<float*>(c->ws + k.logits);
  c->part = reinterpret_cast<float*>(c->ws + k.part);
  c->dxg = reinterpret_cast<float*>(c->ws + k.dxg);
  c->colsum = reinterpret_cast<float*>(c->ws + k.colsum);
  c->tot = reinterpret_cast<int*>(c->ws + k.tot);
  c->colpart = reinterpret_cast<float*>(c->ws + k.colpart);
  c->ep_counts = reinterpret_cast<int*>(c->ws + k.ep_counts);
  c->ep_off = reinterpret_cast<int*>(c->ws + k.ep_off);
  c->ep_tot = reinterpret_cast<int*>(c->ws + k.ep_tot);
  c->gate_scratch = c->ws + k.gate_scratch;
  c->rq = reinterpret_cast<int*>(c->ws + k.rq);
  c->tok_off = reinterpret_cast<int*>(c->ws + k.tok_off);
  c->biasf = reinterpret_cast<float*>(c->ws + k.biasf);
  c->db2part = reinterpret_cast<float*>(c->ws + k.db2part);
  c->ep2_scr = reinterpret_cast<int*>(c->ws + k.ep2_scr);
  c->ep2_base = reinterpret_cast<int*>(c->ws + k.ep2_base);
  c->db2_S = db2_splits(c);
}

}  // namespace moe

extern "C" {

const char* moe_last_error(void) { return g_err.c_str(); }
int moe_abi_version(void) { return MOE_ABI_VERSION; }

int moe_create(moe_ctx** out, int T, int d_model, int d_ff, int E, int dtype, void* nccl_comm,
               int rank, int world) {
  if (!out) return fail(MOE_EINVAL, "moe_create: out is NULL");
  *out = nullptr;
  if (dtype != MOE_F32 && dtype != MOE_BF16) return fail(MOE_EDTYPE, "moe_create: unknown dtype %d", dtype);
  // 16-byte rows for the routing vectors and TMA strides: multiples of 8 (bf16) / 4 (fp32); the
  // tensor-core GEMMs need multiples of 64 (their 64-wide K boxes), other bf16 shapes run the
  // CUDA-core GEMMs (use_tc below)
  const int q = dtype == MOE_BF16 ? 8 : 4;
  if (T < 0 || E < 1 || d_model < 1 || d_ff < 1 || world < 1 || rank < 0 || rank >= world)
    return fail(MOE_ESHAPE, "moe_create: bad dims T=%d E=%d d_model=%d d_ff=%d rank=%d world=%d", T, E,
                d_model, d_ff, rank, world);
  if (E % world != 0)
    return fail(MOE_ESHAPE, "moe_create: E=%d not divisible by world=%d", E, world);
  if (d_model % q != 0 || d_ff % q != 0)
    return fail(MOE_ESHAPE, "moe_create: d_model=%d and d_ff=%d must be multiples of %d for %s", d_model,
                d_ff, q, dtype == MOE_BF16 ? "bf16" : "f32");
  if (E > 128) return fail(MOE_ESHAPE, "moe_create: E=%d > 128 is not supported", E);
  if (world > 1 && !nccl_comm) return fail(MOE_EINVAL, "moe_create: world=%d needs an NCCL comm", world);
  // (world == 1 with a comm enables the EP exchange path against itself: used by the tests)
  moe_ctx* c = new (std::nothrow) moe_ctx();
  if (!c) return fail(MOE_EINVAL, "moe_create: out of host memory");
  c->T = T; c->d = d_model; c->f = d_ff; c->E = E; c->E_local = E / world; c->dtype = dtype;
  c->rank = rank; c->world = world; c->comm = nccl_comm;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  c->sm_count = sms > 0 ? sms : 148;
  c->nblk = (T + moe::kGateBT - 1) / moe::kGateBT;
  c->dwg_splits = T >= 4096 ? 32 : 1;
  c->dwg_splits_max = 64;
  {
    const char* g = getenv("MOE_GEMM");
    c->use_tc = (dtype == MOE_BF16) && !(g && strcmp(g, "simt") == 0) && d_model % 64 == 0 && d_ff % 64 == 0;
  }
  *out = c;
  return MOE_OK;
}

int moe_destroy(moe_ctx* ctx) {
  if (ctx) delete ctx->ep;
  delete ctx;
  return MOE_OK;
}

size_t moe_workspace_bytes(const moe_ctx* ctx) { return ctx ? moe::workspace_bytes(ctx) : 0; }

int moe_set_workspace(moe_ctx* ctx, void* dev_ptr, size_t bytes) {
  if (!ctx) return fail(MOE_EINVAL, "moe_set_workspace: ctx is NULL");
  if (!dev_ptr) return fail(MOE_EINVAL, "moe_set_workspace: dev_ptr is NULL");
  if (reinterpret_cast<uintptr_t>(dev_ptr) % 256 != 0)
    return fail(MOE_EINVAL, "moe_set_workspace: workspace must be 256-byte aligned");
  size_t need = moe::workspace_bytes(ctx);
  if (bytes < need)
    return fail(MOE_EWORKSPACE, "moe_set_workspace: %zu bytes given, %zu needed", bytes, need);
  ctx->ws = reinterpret_cast<uint8_t*>(dev_ptr);
  ctx->ws_bytes = bytes;
  moe::carve_workspace(ctx);
  const int tok_off[2] = {0, (ctx->T + moe::kRowAlign - 1) / moe::kRowAlign * moe::kRowAlign};
  cudaError_t e = cudaMemcpy(ctx->tok_off, tok_off, sizeof(tok_off), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(ctx->flags, 0, 16 * sizeof(int));
  return cuda_status(e, "moe_set_workspace");
}

int moe_check(moe_ctx* ctx, void* stream) {
  int rc = check_ctx(ctx, "moe_check");
  if (rc) return rc;
  int h[4] = {0, 0, 0, 0};
  cudaError_t e = cudaMemcpyAsync(h, ctx->flags, sizeof(h), cudaMemcpyDeviceToHost, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
  if (e != cudaSuccess) return cuda_status(e, "moe_check");
  e = cudaMemsetAsync(ctx->flags, 0, 16 * sizeof(int), S(stream));
  if (e != cudaSuccess) return cuda_status(e, "moe_check");
  if (h[0] & moe::kFlagNonFinite)
    return fail(MOE_ENONFINITE, "moe_check: non-finite gate logit detected (first token %d)", h[1]);
  if (h[0] & moe::kFlagCapacity)
    return fail(MOE_ECAPACITY, "moe_check: R_pad=%d exceeds R_cap; rows beyond R_cap were dropped", h[2]);
  if (h[0] & moe::kFlagArrival)
    return fail(MOE_EARRIVAL, "moe_check: an expert's rows did not all arrive (overlap wait timed out)");
  return MOE_OK;
}

int moe_dts_spawn(moe_ctx* ctx, const void* W1s, const void* b1s, const void* W2s, const void* b2s,
                  const uint32_t* M1bits, const uint32_t* M2bits, void* W1, void* b1, void* W2,
                  void* b2, void* stream) {
  if (!ctx) return fail(MOE_EINVAL, "moe_dts_spawn: ctx is NULL");
  REQUIRE(W1s); REQUIRE(b1s); REQUIRE(W2s); REQUIRE(b2s); REQUIRE(M1bits); REQUIRE(M2bits);
  REQUIRE(W1); REQUIRE(b1); REQUIRE(W2); REQUIRE(b2);
  return cuda_status(moe::launch_spawn(ctx, W1s, b1s, W2s, b2s, M1bits, M2bits, W1, b1, W2, b2, S(stream)),
                     "moe_dts_spawn");
}

int moe_dts_gate(moe_ctx* ctx, const void* x, const void* Wg, const float* u, float tau, float threshold,
                 int top1, float* probs, int32_t* slot, int32_t* counts, int32_t* near_band,
                 void* stream) {
  int rc = check_ctx(ctx, "moe_dts_gate");
  if (rc) return rc;
  REQUIRE_T(x); REQUIRE(Wg); REQUIRE_T(probs); REQUIRE_T(slot); REQUIRE(counts); REQUIRE(near_band);
  if (!(tau > 0.0f) || !isfinite(tau)) return fail(MOE_EINVAL, "moe_dts_gate: tau=%g must be finite and > 0", tau);
  if (!(threshold >= 0.0f && threshold < 1.0f))
    return fail(MOE_EINVAL, "moe_dts_gate: threshold=%g must be in [0, 1)", threshold);
  rc = cuda_status(moe::launch_gate(ctx, x, Wg, u, tau, threshold, top1, probs, slot, counts, near_band, S(stream)),
                   "moe_dts_gate");
  // the per-block expert counts this call left in the workspace belong to (probs, slot)
  ctx->gate_probs = rc == MOE_OK ? probs : nullptr;
  ctx->gate_slot = rc == MOE_OK ? slot : nullptr;
  ++ctx->gate_seq;
  return rc;
}

// moe_dispatch / moe_ep2(d)_dispatch read the per-block expert counts moe_dts_gate left in the
// workspace: accept only the (probs, slot) pair of the most recent moe_dts_gate on this ctx
static int check_gate_outputs(const moe_ctx* ctx, const float* probs, const int32_t* slot, const char* fn) {
  if (ctx->T == 0) return MOE_OK;
  if (ctx->gate_seq == 0)
    return fail(MOE_EINVAL, "%s: no moe_dts_gate has run on this ctx (its per-block counts are needed)", fn);
  if ((const void*)probs != ctx->gate_probs || (const void*)slot != ctx->gate_slot)
    return fail(MOE_EINVAL, "%s: probs/slot are not the outputs of the most recent moe_dts_gate on this ctx "
                "(gate call #%llu)", fn, (unsigned long long)ctx->gate_seq);
  return MOE_OK;
}

int moe_dispatch(moe_ctx* ctx, const void* x, const float* probs, int32_t* slot, void* x_perm,
                 int32_t* row_token, float* row_gate, int32_t* offsets, int64_t R_cap, int32_t* R_out,
                 void* stream) {
  int rc = check_ctx(ctx, "moe_dispatch");
  if (rc) return rc;
  REQUIRE_T(x); REQUIRE_T(probs); REQUIRE_T(slot); REQUIRE_R(x_perm); REQUIRE_R(row_token); REQUIRE_R(row_gate);
  REQUIRE(offsets); REQUIRE(R_out);
  if (R_cap < 0 || R_cap > (int64_t)INT32_MAX) return fail(MOE_EINVAL, "moe_dispatch: bad R_cap %lld", (long long)R_cap);
  if ((rc = check_gate_outputs(ctx, probs, slot, "moe_dispatch"))) return rc;
  return cuda_status(moe::launch_dispatch(ctx, x, probs, slot, nullptr, x_perm, row_token, row_gate,
                                          offsets, R_cap, R_out, S(stream)),
                     "moe_dispatch");
}

int moe_expert_ffn(moe_ctx* ctx, const void* x_perm, const int32_t* offsets, int64_t R_cap, const void* W1,
                   const void* b1, const void* W2, const void* b2, void* gp_saved, void* h_saved,
                   void* e_out, void* stream) {
  int rc = check_ctx(ctx, "moe_expert_ffn");
  if (rc) return rc;
  REQUIRE_R(x_perm); REQUIRE(offsets); REQUIRE(W1); REQUIRE(b1); REQUIRE(W2); REQUIRE(b2);
  REQUIRE_R(h_saved); REQUIRE_R(e_out);      // gp_saved may be NULL (recompute mode)
  if (R_cap < 0 || R_cap % moe::kRowAlign != 0)
    return fail(MOE_EINVAL, "moe_expert_ffn: R_cap=%lld must be a non-negative multiple of %d",
                (long long)R_cap, moe::kRowAlign);
  return cuda_status(moe::launch_expert_ffn(ctx, x_perm, offsets, R_cap, W1, b1, W2, b2, gp_saved, h_saved,
                                            e_out, S(stream)),
                     "moe_expert_ffn");
}

int moe_expert_ffn_recompute(moe_ctx* ctx, const void* x_perm, const int32_t* offsets, int64_t R_cap,
                             const void* W1, const void* b1, void* gp_saved, void* h_saved, void* stream) {
  int rc = check_ctx(ctx, "moe_expert_ffn_recompute");
  if (rc) return rc;
  REQUIRE_R(x_perm); REQUIRE(offsets); REQUIRE(W1); REQUIRE(b1); REQUIRE_R(gp_saved); REQUIRE_R(h_saved);
  if (R_cap < 0 || R_cap % moe::kRowAlign != 0)
    return fail(MOE_EINVAL, "moe_expert_ffn_recompute: R_cap=%lld must be a non-negative multiple of %d",
                (long long)R_cap, moe::kRowAlign);
  return cuda_status(moe::launch_expert_ffn(ctx, x_perm, offsets, R_cap, W1, b1, nullptr, nullptr, gp_saved, h_saved,
                                            nullptr, S(stream)),
                     "moe_expert_ffn_recompute");
}

int moe_combine(moe_ctx* ctx, const void* e_out, const float* row_gate, const int32_t* slot, void* y,
                void* stream) {
  int rc = check_ctx(ctx, "moe_combine");
  if (rc) return rc;
  if (ctx->T == 0) return MOE_OK;
  REQUIRE(e_out); REQUIRE(row_gate); REQUIRE(slot); REQUIRE(y);
  return cuda_status(moe::launch_combine(ctx, e_out, row_gate, slot, y, S(stream)), "moe_combine");
}

int moe_combine_bwd(moe_ctx* ctx, const void* dy, const void* e_out, const float* row_gate,
                    const int32_t* row_token, const int32_t* offsets, int64_t R_cap, void* d_eout,
                    float* dG_row, float* db2, void* stream) {
  int rc = check_ctx(ctx, "moe_combine_bwd");
  if (rc) return rc;
  REQUIRE_T(dy); REQUIRE_R(e_out); REQUIRE_R(row_gate); REQUIRE_R(row_token); REQUIRE(offsets); REQUIRE_R(d_eout);
  REQUIRE_R(dG_row);
  if (R_cap < 0) return fail(MOE_EINVAL, "moe_combine_bwd: bad R_cap");
  if (db2 && (ctx->comm || ctx->world > 1))
    return fail(MOE_EINVAL, "moe_combine_bwd: db2 is an expert-side sum; under the NCCL exchange it comes from "
                "moe_expert_ffn_bwd on the received d_eout");
  return cuda_status(moe::launch_combine_bwd(ctx, dy, e_out, row_gate, row_token, offsets, R_cap, d_eout,
                                             dG_row, db2, S(stream)),
                     "moe_combine_bwd");
}

int moe_expert_ffn_bwd(moe_ctx* ctx, const void* d_eout, const void* x_perm, const void* gp_saved,
                       const void* h_saved, const int32_t* offsets, int64_t R_cap, const void* W1,
                       const void* W2, void* da, void* dx_perm, float* dW1, float* db1, float* dW2,
                       float* db2, void* stream) {
  int rc = check_ctx(ctx, "moe_expert_ffn_bwd");
  if (rc) return rc;
  REQUIRE_R(d_eout); REQUIRE_R(x_perm); REQUIRE_R(gp_saved); REQUIRE_R(h_saved); REQUIRE(offsets); REQUIRE(W1);
  REQUIRE(W2); REQUIRE_R(da); REQUIRE_R(dx_perm); REQUIRE(dW1); REQUIRE(db1); REQUIRE(dW2);   // db2 optional
  if (R_cap < 0 || R_cap % moe::kRowAlign != 0)
    return fail(MOE_EINVAL, "moe_expert_ffn_bwd: R_cap=%lld must be a non-negative multiple of %d",
                (long long)R_cap, moe::kRowAlign);
  return cuda_status(moe::launch_expert_ffn_bwd(ctx, d_eout, x_perm, gp_saved, h_saved, offsets, R_cap, W1,
                                                W2, da, dx_perm, dW1, db1, dW2, db2, S(stream)),
                     "moe_expert_ffn_bwd");
}

int moe_dts_gate_bwd(moe_ctx* ctx, const float* dG_row, const int32_t* slot, const float* probs,
                     const void* x, const void* Wg, float tau, float balance_alpha, const int32_t* counts,
                     int64_t B_total, float* dWg, float* dlogits, void* dx, void* stream) {
  int rc = check_ctx(ctx, "moe_dts_gate_bwd");
  if (rc) return rc;
  REQUIRE(dG_row); REQUIRE_T(slot); REQUIRE_T(probs); REQUIRE_T(x); REQUIRE(dWg); REQUIRE_T(dlogits);
  if (dx && !Wg) return fail(MOE_EINVAL, "moe_dts_gate_bwd: dx (dlogits W_g^T) requested without Wg");
  if (!(tau > 0.0f) || !isfinite(tau)) return fail(MOE_EINVAL, "moe_dts_gate_bwd: tau=%g must be finite and > 0", tau);
  if (!(balance_alpha >= 0.0f) || !isfinite(balance_alpha))
    return fail(MOE_EINVAL, "moe_dts_gate_bwd: balance_alpha=%g must be finite and >= 0", balance_alpha);
  if (balance_alpha > 0.0f && (!counts || B_total <= 0))
    return fail(MOE_EINVAL, "moe_dts_gate_bwd: balance term needs counts and B_total > 0");
  return cuda_status(moe::launch_gate_bwd(ctx, dG_row, slot, probs, x, Wg, tau, balance_alpha, counts, 1, B_total,
                                          dWg, dlogits, dx, S(stream)),
                     "moe_dts_gate_bwd");
}

int moe_dispatch_bwd(moe_ctx* ctx, const void* dx_perm, const int32_t* slot, int accumulate, void* dx,
                     void* stream) {
  int rc = check_ctx(ctx, "moe_dispatch_bwd");
  if (rc) return rc;
  REQUIRE(dx_perm); REQUIRE_T(slot); REQUIRE_T(dx);
  return cuda_status(moe::launch_dispatch_bwd(ctx, dx_perm, slot, accumulate, dx, S(stream)), "moe_dispatch_bwd");
}

int moe_balance_loss(moe_ctx* ctx, const float* probs, const int32_t* counts, float alpha, int64_t B_total,
                     float* loss, void* stream) {
  int rc = check_ctx(ctx, "moe_balance_loss");
  if (rc) return rc;
  REQUIRE_T(probs); REQUIRE(counts); REQUIRE(loss);
  if (B_total <= 0) return fail(MOE_EINVAL, "moe_balance_loss: B_total must be > 0");
  return cuda_status(moe::launch_balance_loss(ctx, probs, counts, alpha, B_total, loss, S(stream)),
                     "moe_balance_loss");
}

}  // extern "C"

#include <atomic>
namespace moe {
static std::atomic<unsigned long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
}  // namespace moe

extern "C" uint64_t moe_kernel_launch_count(void) { return moe::g_launches.load(); }

// ====================================================================== expert parallelism
namespace {
#ifdef MOE_HAVE_NCCL
int nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return MOE_OK;
  return fail(MOE_ENCCL, "%s: NCCL error %d (%s)", where, (int)r, ncclGetErrorString(r));
}
#endif
int check_ep(moe_ctx* c, const char* fn, bool need_plan) {
  if (!c) return fail(MOE_EINVAL, "%s: ctx is NULL", fn);
  if (!c->comm) return fail(MOE_EINVAL, "%s: ctx has no NCCL communicator (expert parallelism disabled)", fn);
  if (c->comm == MOE_COMM_EMULATED && !need_plan)
    return fail(MOE_EINVAL, "%s: needs a real NCCL communicator (ctx is a single-process emulated rank)", fn);
  if (need_plan && !c->ep) return fail(MOE_EINVAL, "%s: no exchange plan (call moe_ep_plan first)", fn);
  return MOE_OK;
}
// the hierarchical exchange relays rows through the caller's staging buffer
int check_stage(moe_ctx* c, const char* fn) {
  if (c->ep->G >= c->world) return MOE_OK;
  const long long need = c->ep->H.stage_out + c->ep->H.stage_in;
  if (need > 0 && (!c->ep_stage || c->ep_stage_rows < need))
    return fail(MOE_ECAPACITY, "%s: hierarchical exchange needs %lld staging rows (moe_ep_set_stage), have %lld", fn,
                need, (long long)c->ep_stage_rows);
  return MOE_OK;
}
}  // namespace

extern "C" {

int moe_nccl_unique_id(void* id_out, size_t bytes) {
#ifdef MOE_HAVE_NCCL
  if (!id_out || bytes < sizeof(ncclUniqueId)) return fail(MOE_EINVAL, "moe_nccl_unique_id: need %zu bytes", sizeof(ncclUniqueId));
  return nccl_status(ncclGetUniqueId(reinterpret_cast<ncclUniqueId*>(id_out)), "moe_nccl_unique_id");
#else
  return fail(MOE_ENCCL, "moe_nccl_unique_id: built without NCCL");
#endif
}

int moe_nccl_comm_init(void** comm_out, const void* id, int world, int rank) {
#ifdef MOE_HAVE_NCCL
  if (!comm_out || !id) return fail(MOE_EINVAL, "moe_nccl_comm_init: NULL argument");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  int rc = nccl_status(ncclCommInitRank(&comm, world, uid, rank), "moe_nccl_comm_init");
  *comm_out = comm;
  return rc;
#else
  return fail(MOE_ENCCL, "moe_nccl_comm_init: built without NCCL");
#endif
}

int moe_nccl_comm_destroy(void* comm) {
#ifdef MOE_HAVE_NCCL
  if (!comm) return MOE_OK;
  return nccl_status(ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)), "moe_nccl_comm_destroy");
#else
  return fail(MOE_ENCCL, "moe_nccl_comm_destroy: built without NCCL");
#endif
}

int moe_ep_plan(moe_ctx* ctx, const int32_t* counts_all, int32_t* offsets_send, int32_t* offsets_recv, int64_t* R_send,
                int64_t* R_recv) {
  if (!ctx) return fail(MOE_EINVAL, "moe_ep_plan: ctx is NULL");
  REQUIRE(counts_all);
  for (long long i = 0; i < (long long)ctx->world * ctx->E; ++i)
    if (counts_all[i] < 0 || counts_all[i] > ctx->T)
      return fail(MOE_EINVAL, "moe_ep_plan: counts_all[%lld]=%d outside [0, T=%d]", i, counts_all[i], ctx->T);
  if (!ctx->ep) ctx->ep = new (std::nothrow) moe::EpPlan();
  if (!ctx->ep) return fail(MOE_EINVAL, "moe_ep_plan: out of host memory");
  moe::ep_build_plan(*ctx->ep, counts_all, ctx->world, ctx->E, ctx->rank);
  const int G = ctx->ep_G > 0 ? ctx->ep_G : ctx->world;
  ctx->ep->G = G;
  if (G < ctx->world) moe::ep_build_hier(ctx->ep->H, counts_all, ctx->world, ctx->E, ctx->rank, G, ctx->ep->offsets_send);
  const moe::EpPlan& P = *ctx->ep;
  if (offsets_send) memcpy(offsets_send, P.offsets_send.data(), sizeof(int) * (ctx->E + 1));
  if (offsets_recv) memcpy(offsets_recv, P.offsets_recv.data(), sizeof(int) * (ctx->E_local + 1));
  if (R_send) *R_send = P.R_send;
  if (R_recv) *R_recv = P.R_recv;
  return MOE_OK;
}

int moe_ep_plan_chunks(moe_ctx* ctx, int which, int32_t* peer, int64_t* row, int32_t* nrows, int max_chunks,
                       int* n_out) {
  if (!ctx || !ctx->ep) return fail(MOE_EINVAL, "moe_ep_plan_chunks: no plan");
  REQUIRE(n_out);
  const moe::EpPlan& P = *ctx->ep;
  const std::vector<int>& pe = which == 0 ? P.s_peer : P.r_peer;
  const std::vector<int>& nr = which == 0 ? P.s_rows : P.r_rows;
  const std::vector<long long>& ro = which == 0 ? P.s_src : P.r_dst;
  *n_out = (int)pe.size();
  for (int i = 0; i < (int)pe.size() && i < max_chunks; ++i) {
    if (peer) peer[i] = pe[i];
    if (row) row[i] = ro[i];
    if (nrows) nrows[i] = nr[i];
  }
  return MOE_OK;
}

int moe_ep_set_topology(moe_ctx* ctx, int gpus_per_node) {
  if (!ctx) return fail(MOE_EINVAL, "moe_ep_set_topology: ctx is NULL");
  if (gpus_per_node <= 0 || ctx->world % gpus_per_node != 0)
    return fail(MOE_EINVAL, "moe_ep_set_topology: gpus_per_node=%d must divide world=%d", gpus_per_node, ctx->world);
  ctx->ep_G = gpus_per_node;
  return MOE_OK;
}

int moe_ep_stage_rows(moe_ctx* ctx, int64_t* rows) {
  if (!ctx || !ctx->ep) return fail(MOE_EINVAL, "moe_ep_stage_rows: no plan");
  REQUIRE(rows);
  *rows = ctx->ep->G < ctx->world ? ctx->ep->H.stage_out + ctx->ep->H.stage_in : 0;
  return MOE_OK;
}

int moe_ep_set_stage(moe_ctx* ctx, void* stage, int64_t rows_cap) {
  if (!ctx) return fail(MOE_EINVAL, "moe_ep_set_stage: ctx is NULL");
  if (rows_cap < 0 || (rows_cap > 0 && !stage)) return fail(MOE_EINVAL, "moe_ep_set_stage: bad buffer");
  ctx->ep_stage = stage;
  ctx->ep_stage_rows = rows_cap;
  return MOE_OK;
}

int moe_ep_hier_chunks(moe_ctx* ctx, int phase, int is_recv, int32_t* peer, int32_t* buf, int64_t* row,
                       int32_t* nrows, int max_chunks, int* n_out) {
  if (!ctx || !ctx->ep) return fail(MOE_EINVAL, "moe_ep_hier_chunks: no plan");
  if (phase < 0 || phase > 2) return fail(MOE_EINVAL, "moe_ep_hier_chunks: phase %d", phase);
  REQUIRE(n_out);
  const std::vector<moe::EpMsg>& v = is_recv ? ctx->ep->H.rcv[phase] : ctx->ep->H.snd[phase];
  *n_out = ctx->ep->G < ctx->world ? (int)v.size() : 0;
  for (int i = 0; i < *n_out && i < max_chunks; ++i) {
    if (peer) peer[i] = v[i].peer;
    if (buf) buf[i] = v[i].buf;
    if (row) row[i] = v[i].row;
    if (nrows) nrows[i] = v[i].rows;
  }
  return MOE_OK;
}

// Host-only cost-model identities of the two exchange plans over a virtual topology
// (world ranks, G per node) for the routing counts_all [world][E]: stats =
// { flat: inter-node (src GPU, dst GPU) pairs with payload, inter-node rows, intra-node rows,
//   hierarchical: inter-node messages, inter-node rows, intra-node rows moved (phases 0 and 2),
//   ordered node pairs with payload, max rows of one inter-node message }.
int moe_ep_topology_stats(int world, int gpus_per_node, int E, const int32_t* counts_all, int64_t* stats) {
  if (world <= 0 || gpus_per_node <= 0 || world % gpus_per_node != 0 || E % world != 0)
    return fail(MOE_EINVAL, "moe_ep_topology_stats: world=%d G=%d E=%d", world, gpus_per_node, E);
  REQUIRE(counts_all); REQUIRE(stats);
  const int G = gpus_per_node, El = E / world;
  for (int i = 0; i < 8; ++i) stats[i] = 0;
  std::vector<char> node_pair((size_t)(world / G) * (world / G), 0);
  for (int q = 0; q < world; ++q)
    for (int p = 0; p < world; ++p) {
      long long n = 0;
      for (int j = 0; j < El; ++j) n += counts_all[(long long)q * E + p * El + j];
      if (q / G != p / G) {
        if (n > 0) { stats[0] += 1; node_pair[(size_t)(q / G) * (world / G) + p / G] = 1; }
        stats[1] += n;
      } else {
        stats[2] += n;
      }
    }
  for (char b : node_pair) stats[6] += b;
  for (int r = 0; r < world; ++r) {
    moe::EpPlan P;
    moe::ep_build_plan(P, counts_all, world, E, r);
    if (G >= world) continue;
    moe::ep_build_hier(P.H, counts_all, world, E, r, G, P.offsets_send);
    for (const moe::EpMsg& m : P.H.snd[1]) {
      stats[3] += 1;
      stats[4] += m.rows;
      if (m.rows > stats[7]) stats[7] = m.rows;
    }
    for (int ph : {0, 2})
      for (const moe::EpMsg& m : P.H.snd[ph]) stats[5] += m.rows;
  }
  if (G >= world) { stats[5] = stats[2]; }
  return MOE_OK;
}

int moe_ep_exchange_counts(moe_ctx* ctx, const int32_t* counts, int32_t* counts_all_host, void* stream) {
  int rc = check_ctx(ctx, "moe_ep_exchange_counts");
  if (rc) return rc;
  if ((rc = check_ep(ctx, "moe_ep_exchange_counts", false))) return rc;
  REQUIRE(counts); REQUIRE(counts_all_host);
#ifdef MOE_HAVE_NCCL
  rc = nccl_status(ncclAllGather(counts, ctx->ep_counts, ctx->E, ncclInt32, reinterpret_cast<ncclComm_t>(ctx->comm),
                                 S(stream)),
                   "moe_ep_exchange_counts");
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(counts_all_host, ctx->ep_counts, sizeof(int) * ctx->world * ctx->E,
                                  cudaMemcpyDeviceToHost, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
  return cuda_status(e, "moe_ep_exchange_counts");
#else
  return fail(MOE_ENCCL, "moe_ep_exchange_counts: built without NCCL");
#endif
}

int moe_ep_upload(moe_ctx* ctx, int32_t* offsets_recv_dev, void* stream) {
  int rc = check_ctx(ctx, "moe_ep_upload");
  if (rc) return rc;
  if ((rc = check_ep(ctx, "moe_ep_upload", true))) return rc;
  if (ctx->comm == MOE_COMM_EMULATED) return fail(MOE_EINVAL, "moe_ep_upload: emulated rank");
  REQUIRE(offsets_recv_dev);
  const moe::EpPlan& P = *ctx->ep;
  cudaError_t e = cudaMemcpyAsync(offsets_recv_dev, P.offsets_recv.data(), sizeof(int) * (ctx->E_local + 1),
                                  cudaMemcpyHostToDevice, S(stream));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ctx->ep_off, P.offsets_recv.data(), sizeof(int) * (ctx->E_local + 1), cudaMemcpyHostToDevice,
                        S(stream));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ctx->ep_tot, P.recv_tot.data(), sizeof(int) * ctx->E_local, cudaMemcpyHostToDevice, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));   // host vectors are pageable
  return cuda_status(e, "moe_ep_upload");
}

int moe_ep_dispatch(moe_ctx* ctx, const void* send_rows, void* recv_rows, int width, int64_t R_recv_cap, void* stream) {
  int rc = check_ctx(ctx, "moe_ep_dispatch");
  if (rc) return rc;
  if ((rc = check_ep(ctx, "moe_ep_dispatch", true))) return rc;
  if (ctx->comm == MOE_COMM_EMULATED) return fail(MOE_EINVAL, "moe_ep_dispatch: emulated rank (use moe_ep2_*)");
  if (width <= 0 || width % 8 != 0) return fail(MOE_ESHAPE, "moe_ep_dispatch: width=%d must be a positive multiple of 8", width);
  if (R_recv_cap < ctx->ep->R_recv)
    return fail(MOE_ECAPACITY, "moe_ep_dispatch: R_recv_cap=%lld < plan R_recv=%lld", (long long)R_recv_cap,
                (long long)ctx->ep->R_recv);
#ifdef MOE_HAVE_NCCL
  if ((rc = check_stage(ctx, "moe_ep_dispatch"))) return rc;
  rc = ctx->ep->G < ctx->world
           ? nccl_status(moe::ep_exchange_hier(ctx, *ctx->ep, send_rows, recv_rows, ctx->ep_stage, width, 0, S(stream)),
                         "moe_ep_dispatch")
           : nccl_status(moe::ep_exchange(ctx, *ctx->ep, send_rows, recv_rows, width, 0, S(stream)), "moe_ep_dispatch");
  if (rc) return rc;
  return cuda_status(moe::launch_zero_pads(ctx, recv_rows, ctx->ep_off, ctx->ep_tot, width, S(stream)), "moe_ep_dispatch");
#else
  return fail(MOE_ENCCL, "moe_ep_dispatch: built without NCCL");
#endif
}

int moe_ep_combine(moe_ctx* ctx, const void* recv_rows, void* send_rows, int width, void* stream) {
  int rc = check_ctx(ctx, "moe_ep_combine");
  if (rc) return rc;
  if ((rc = check_ep(ctx, "moe_ep_combine", true))) return rc;
  if (ctx->comm == MOE_COMM_EMULATED) return fail(MOE_EINVAL, "moe_ep_combine: emulated rank (use moe_ep2_*)");
  if (width <= 0 || width % 8 != 0) return fail(MOE_ESHAPE, "moe_ep_combine: width=%d must be a positive multiple of 8", width);
#ifdef MOE_HAVE_NCCL
  if ((rc = check_stage(ctx, "moe_ep_combine"))) return rc;
  if (ctx->ep->G < ctx->world)
    return nccl_status(moe::ep_exchange_hier(ctx, *ctx->ep, recv_rows, send_rows, ctx->ep_stage, width, 1, S(stream)),
                       "moe_ep_combine");
  return nccl_status(moe::ep_exchange(ctx, *ctx->ep, recv_rows, send_rows, width, 1, S(stream)), "moe_ep_combine");
#else
  return fail(MOE_ENCCL, "moe_ep_combine: built without NCCL");
#endif
}

int moe_ep_allreduce(moe_ctx* ctx, void* buf, int64_t n, int is_int32, void* stream) {
  int rc = check_ctx(ctx, "moe_ep_allreduce");
  if (rc) return rc;
  if ((rc = check_ep(ctx, "moe_ep_allreduce", false))) return rc;
  REQUIRE(buf);
#ifdef MOE_HAVE_NCCL
  return nccl_status(ncclAllReduce(buf, buf, (size_t)n, is_int32 ? ncclInt32 : ncclFloat32, ncclSum,
                                   reinterpret_cast<ncclComm_t>(ctx->comm), S(stream)),
                     "moe_ep_allreduce");
#else
  return fail(MOE_ENCCL, "moe_ep_allreduce: built without NCCL");
#endif
}

}  // extern "C"

// ====================================================================== fused peer-memory EP (ep2)
namespace {
int ep2_check(moe_ctx* c, const char* fn) {
  int rc = check_ctx(c, fn);
  if (rc) return rc;
  if (!c->comm) return fail(MOE_EINVAL, "%s: ctx has no communicator (expert parallelism disabled)", fn);
  if (c->world > moe::kMaxPeers) return fail(MOE_ESHAPE, "%s: world=%d > %d", fn, c->world, moe::kMaxPeers);
  return MOE_OK;
}
int ep2_table(moe_ctx* c, const void* const* peers, moe::PeerTable& t, const char* fn) {
  if (!peers) return fail(MOE_EINVAL, "%s: peer pointer array is NULL", fn);
  t = moe::PeerTable{};
  for (int i = 0; i < c->world; ++i) {
    if (!peers[i]) return fail(MOE_EINVAL, "%s: peer pointer %d is NULL", fn, i);
    t.p[i] = peers[i];
  }
  return MOE_OK;
}
}  // namespace

extern "C" {

int moe_ep2_barrier(moe_ctx* ctx, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_barrier");
  if (rc) return rc;
  if (ctx->comm == MOE_COMM_EMULATED || ctx->world == 1) return MOE_OK;
#ifdef MOE_HAVE_NCCL
  // stream-ordered barrier: a 1-element all-reduce completes only when every rank reached it
  return nccl_status(ncclAllReduce(ctx->flags + 8, ctx->flags + 8, 1, ncclInt32, ncclSum,
                                   reinterpret_cast<ncclComm_t>(ctx->comm), S(stream)),
                     "moe_ep2_barrier");
#else
  return fail(MOE_ENCCL, "moe_ep2_barrier: built without NCCL");
#endif
}

int moe_ep2_counts(moe_ctx* ctx, const int32_t* counts, int32_t* const* counts_all_peers, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_counts");
  if (rc) return rc;
  REQUIRE(counts);
  moe::PeerTable t;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(counts_all_peers), t, "moe_ep2_counts"))) return rc;
  return cuda_status(moe::launch_ep2_counts(ctx, counts, t, S(stream)), "moe_ep2_counts");
}

int moe_ep2_plan(moe_ctx* ctx, const int32_t* counts_all, int64_t R_recv_cap, int32_t* offsets_recv, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_plan");
  if (rc) return rc;
  REQUIRE(counts_all);
  if (R_recv_cap < 0) return fail(MOE_EINVAL, "moe_ep2_plan: bad R_recv_cap");
  return cuda_status(moe::launch_ep2_plan(ctx, counts_all, R_recv_cap, offsets_recv, S(stream)), "moe_ep2_plan");
}

int moe_ep2_prepare_recv(moe_ctx* ctx, void* x_recv, int32_t* rtok, int32_t* rsrc, float* rgate, int64_t R_recv_cap,
                         void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_prepare_recv");
  if (rc) return rc;
  REQUIRE(x_recv); REQUIRE(rtok); REQUIRE(rsrc); REQUIRE(rgate);
  return cuda_status(moe::launch_ep2_prepare(ctx, x_recv, rtok, rsrc, rgate, R_recv_cap, S(stream)),
                     "moe_ep2_prepare_recv");
}

int moe_ep2_dispatch(moe_ctx* ctx, const void* x, const float* probs, int32_t* slot, void* const* x_recv_peers,
                     int32_t* const* rtok_peers, int32_t* const* rsrc_peers, float* const* rgate_peers,
                     int64_t R_recv_cap, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_dispatch");
  if (rc) return rc;
  REQUIRE_T(x); REQUIRE_T(probs); REQUIRE_T(slot);
  if ((rc = check_gate_outputs(ctx, probs, slot, "moe_ep2_dispatch"))) return rc;
  moe::PeerTable xr, rt, rs, rg;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(x_recv_peers), xr, "moe_ep2_dispatch")) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rtok_peers), rt, "moe_ep2_dispatch")) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rsrc_peers), rs, "moe_ep2_dispatch")) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rgate_peers), rg, "moe_ep2_dispatch")))
    return rc;
  return cuda_status(moe::launch_ep2_dispatch(ctx, x, probs, slot, xr, rt, rs, rg, R_recv_cap, S(stream)),
                     "moe_ep2_dispatch");
}

int moe_ep2_arrival_plan(moe_ctx* ctx, const int32_t* counts_all, int32_t* sprefix, int32_t* arrive_target,
                         void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_arrival_plan");
  if (rc) return rc;
  REQUIRE(counts_all); REQUIRE(sprefix); REQUIRE(arrive_target);
  return cuda_status(moe::launch_ep2_arrival_plan(ctx, counts_all, sprefix, arrive_target, S(stream)),
                     "moe_ep2_arrival_plan");
}

int moe_ep2_dispatch_ordered(moe_ctx* ctx, const void* x, const float* probs, int32_t* slot, void* const* x_recv_peers,
                             int32_t* const* rtok_peers, int32_t* const* rsrc_peers, float* const* rgate_peers,
                             int64_t R_recv_cap, const int32_t* sprefix, int32_t* send, int32_t* const* arrive_peers,
                             void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_dispatch_ordered");
  if (rc) return rc;
  REQUIRE_T(x); REQUIRE_T(probs); REQUIRE_T(slot); REQUIRE(sprefix);
  if (ctx->T > 0 && !send) return fail(MOE_EINVAL, "moe_ep2_dispatch_ordered: send is NULL");
  if ((rc = check_gate_outputs(ctx, probs, slot, "moe_ep2_dispatch_ordered"))) return rc;
  moe::PeerTable xr, rt, rs, rg, ar;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(x_recv_peers), xr, "moe_ep2_dispatch_ordered")) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rtok_peers), rt, "moe_ep2_dispatch_ordered")) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rsrc_peers), rs, "moe_ep2_dispatch_ordered")) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rgate_peers), rg, "moe_ep2_dispatch_ordered")) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(arrive_peers), ar, "moe_ep2_dispatch_ordered")))
    return rc;
  return cuda_status(moe::launch_ep2_dispatch(ctx, x, probs, slot, xr, rt, rs, rg, R_recv_cap, S(stream), sprefix,
                                              send, &ar),
                     "moe_ep2_dispatch_ordered");
}

int moe_ep2_expert_ffn(moe_ctx* ctx, const void* x_recv, const int32_t* offsets_recv, int64_t R_recv_cap,
                       const void* W1, const void* b1, const void* W2, const void* b2, void* gp_saved, void* h_saved,
                       void* e_out, const int32_t* arrive, const int32_t* arrive_target, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_expert_ffn");
  if (rc) return rc;
  const int64_t R_cap = R_recv_cap;
  REQUIRE_R(x_recv); REQUIRE(offsets_recv); REQUIRE(W1); REQUIRE(b1); REQUIRE(W2); REQUIRE(b2);
  REQUIRE_R(h_saved); REQUIRE_R(e_out); REQUIRE(arrive); REQUIRE(arrive_target);
  if (R_recv_cap < 0 || R_recv_cap % moe::kRowAlign != 0)
    return fail(MOE_EINVAL, "moe_ep2_expert_ffn: R_recv_cap=%lld must be a non-negative multiple of %d",
                (long long)R_recv_cap, moe::kRowAlign);
  return cuda_status(moe::launch_expert_ffn(ctx, x_recv, offsets_recv, R_recv_cap, W1, b1, W2, b2, gp_saved, h_saved,
                                            e_out, S(stream), arrive, arrive_target),
                     "moe_ep2_expert_ffn");
}

int moe_ep2_combine(moe_ctx* ctx, void* const* e_out_peers, const float* probs, const int32_t* slot, void* y,
                    void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_combine");
  if (rc) return rc;
  REQUIRE_T(probs); REQUIRE_T(slot); REQUIRE_T(y);
  moe::PeerTable t;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(e_out_peers), t, "moe_ep2_combine"))) return rc;
  return cuda_status(moe::launch_ep2_combine(ctx, t, probs, slot, y, S(stream)), "moe_ep2_combine");
}

int moe_ep2_combine_bwd(moe_ctx* ctx, void* const* dy_peers, const void* e_out, const float* rgate,
                        const int32_t* rtok, const int32_t* rsrc, const int32_t* offsets_recv, int64_t R_recv_cap,
                        void* d_eout, float* dG_row, float* db2, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_combine_bwd");
  if (rc) return rc;
  REQUIRE(e_out); REQUIRE(rgate); REQUIRE(rtok); REQUIRE(rsrc); REQUIRE(offsets_recv); REQUIRE(d_eout); REQUIRE(dG_row);
  moe::PeerTable t;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(dy_peers), t, "moe_ep2_combine_bwd"))) return rc;
  return cuda_status(moe::launch_ep2_combine_bwd(ctx, t, e_out, rgate, rtok, rsrc, offsets_recv, R_recv_cap, d_eout,
                                                 dG_row, db2, S(stream)),
                     "moe_ep2_combine_bwd");
}

int moe_ep2_gate_bwd(moe_ctx* ctx, float* const* dG_peers, const int32_t* slot, const float* probs, const void* x,
                     const void* Wg, float tau, float balance_alpha, const int32_t* counts_all, int64_t B_total,
                     float* dWg, float* dlogits, void* dx, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_gate_bwd");
  if (rc) return rc;
  REQUIRE_T(slot); REQUIRE_T(probs); REQUIRE_T(x); REQUIRE(dWg); REQUIRE_T(dlogits);
  if (dx && !Wg) return fail(MOE_EINVAL, "moe_ep2_gate_bwd: dx (dlogits W_g^T) requested without Wg");
  const int32_t* counts = counts_all;
  if (!(tau > 0.0f) || !isfinite(tau)) return fail(MOE_EINVAL, "moe_ep2_gate_bwd: tau=%g must be finite and > 0", tau);
  if (!(balance_alpha >= 0.0f) || !isfinite(balance_alpha))
    return fail(MOE_EINVAL, "moe_ep2_gate_bwd: balance_alpha=%g must be finite and >= 0", balance_alpha);
  if (balance_alpha > 0.0f && (!counts || B_total <= 0))
    return fail(MOE_EINVAL, "moe_ep2_gate_bwd: balance term needs counts and B_total > 0");
  moe::PeerTable t;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(dG_peers), t, "moe_ep2_gate_bwd"))) return rc;
  // counts_all [world][E]: the kernel sums the world rows -> the global counts of Eq. 10
  return cuda_status(moe::launch_gate_bwd_peer(ctx, t, slot, probs, x, Wg, tau, balance_alpha, counts, ctx->world,
                                               B_total, dWg, dlogits, dx, S(stream)),
                     "moe_ep2_gate_bwd");
}

int moe_ep2_dispatch_bwd(moe_ctx* ctx, void* const* dx_perm_peers, const int32_t* slot, int accumulate, void* dx,
                         void* stream) {
  int rc = ep2_check(ctx, "moe_ep2_dispatch_bwd");
  if (rc) return rc;
  REQUIRE_T(slot); REQUIRE_T(dx);
  moe::PeerTable t;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(dx_perm_peers), t, "moe_ep2_dispatch_bwd"))) return rc;
  return cuda_status(moe::launch_ep2_dispatch_bwd(ctx, t, slot, accumulate, dx, S(stream)), "moe_ep2_dispatch_bwd");
}

// ---------------------------------------------------------------- ep2 with token dedup
int moe_ep2d_dispatch(moe_ctx* ctx, const void* x, const float* probs, int32_t* slot, int32_t* uslot,
                      void* const* tokbuf_peers, int32_t* const* urows_peers, int32_t* const* rtok_peers,
                      int32_t* const* rsrc_peers, float* const* rgate_peers, int32_t* const* ruid_peers,
                      int64_t R_recv_cap, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2d_dispatch");
  if (rc) return rc;
  REQUIRE_T(x); REQUIRE_T(probs); REQUIRE_T(slot); REQUIRE_T(uslot);
  if ((rc = check_gate_outputs(ctx, probs, slot, "moe_ep2d_dispatch"))) return rc;
  if ((long long)ctx->world * ctx->T > 0x7fffffffLL) return fail(MOE_ESHAPE, "moe_ep2d_dispatch: world*T exceeds int32");
  moe::PeerTable tb, ur, rt, rs, rg, ru;
  const char* fn = "moe_ep2d_dispatch";
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(tokbuf_peers), tb, fn)) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(urows_peers), ur, fn)) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rtok_peers), rt, fn)) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rsrc_peers), rs, fn)) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(rgate_peers), rg, fn)) ||
      (rc = ep2_table(ctx, reinterpret_cast<const void* const*>(ruid_peers), ru, fn)))
    return rc;
  return cuda_status(moe::launch_ep2d_dispatch(ctx, x, probs, slot, uslot, tb, ur, rt, rs, rg, ru, R_recv_cap,
                                               S(stream)), fn);
}

int moe_ep2d_permute(moe_ctx* ctx, const void* tokbuf, const int32_t* rtok, int32_t* ruid, int64_t R_recv_cap,
                     void* x_recv, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2d_permute");
  if (rc) return rc;
  REQUIRE(tokbuf); REQUIRE(rtok); REQUIRE(ruid); REQUIRE(x_recv);
  if (R_recv_cap < 0) return fail(MOE_EINVAL, "moe_ep2d_permute: bad R_recv_cap");
  return cuda_status(moe::launch_ep2d_permute(ctx, tokbuf, rtok, ruid, R_recv_cap, x_recv, S(stream)),
                     "moe_ep2d_permute");
}

int moe_ep2d_presum(moe_ctx* ctx, const void* rows, const float* rgate_or_null, const int32_t* urows, void* out,
                    void* stream) {
  int rc = ep2_check(ctx, "moe_ep2d_presum");
  if (rc) return rc;
  REQUIRE(rows); REQUIRE(urows); REQUIRE(out);
  return cuda_status(moe::launch_ep2d_presum(ctx, rows, rgate_or_null, urows, out, S(stream)), "moe_ep2d_presum");
}

int moe_ep2d_gather_dy(moe_ctx* ctx, void* const* dy_peers, const int32_t* urows, void* dyu, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2d_gather_dy");
  if (rc) return rc;
  REQUIRE(urows); REQUIRE(dyu);
  moe::PeerTable t;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(dy_peers), t, "moe_ep2d_gather_dy"))) return rc;
  return cuda_status(moe::launch_ep2d_gather_dy(ctx, t, urows, dyu, S(stream)), "moe_ep2d_gather_dy");
}

int moe_ep2d_combine(moe_ctx* ctx, void* const* ysum_peers, const int32_t* uslot, void* y, void* stream) {
  int rc = ep2_check(ctx, "moe_ep2d_combine");
  if (rc) return rc;
  REQUIRE_T(uslot); REQUIRE_T(y);
  moe::PeerTable t;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(ysum_peers), t, "moe_ep2d_combine"))) return rc;
  return cuda_status(moe::launch_ep2d_combine(ctx, t, uslot, y, S(stream)), "moe_ep2d_combine");
}

int moe_ep2d_combine_bwd(moe_ctx* ctx, const void* dyu, const void* e_out, const float* rgate, const int32_t* ruid,
                         const int32_t* offsets_recv, int64_t R_recv_cap, void* d_eout, float* dG_row, float* db2,
                         void* stream) {
  int rc = ep2_check(ctx, "moe_ep2d_combine_bwd");
  if (rc) return rc;
  REQUIRE(dyu); REQUIRE(e_out); REQUIRE(rgate); REQUIRE(ruid); REQUIRE(offsets_recv); REQUIRE(d_eout); REQUIRE(dG_row);
  return cuda_status(moe::launch_ep2d_combine_bwd(ctx, dyu, e_out, rgate, ruid, offsets_recv, R_recv_cap, d_eout,
                                                  dG_row, db2, S(stream)),
                     "moe_ep2d_combine_bwd");
}

int moe_ep2d_dispatch_bwd(moe_ctx* ctx, void* const* dxu_peers, const int32_t* uslot, int accumulate, void* dx,
                          void* stream) {
  int rc = ep2_check(ctx, "moe_ep2d_dispatch_bwd");
  if (rc) return rc;
  REQUIRE_T(uslot); REQUIRE_T(dx);
  moe::PeerTable t;
  if ((rc = ep2_table(ctx, reinterpret_cast<const void* const*>(dxu_peers), t, "moe_ep2d_dispatch_bwd"))) return rc;
  return cuda_status(moe::launch_ep2_dispatch_bwd(ctx, t, uslot, accumulate, dx, S(stream), ctx->world, 1),
                     "moe_ep2d_dispatch_bwd");
}

}  // extern "C"
