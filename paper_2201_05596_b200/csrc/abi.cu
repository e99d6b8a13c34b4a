// extern "C" entry points of libmoe_b200.so (declared in include/moe_b200.h).
// Arguments are validated here, before any launch, so a bad call returns
// MOE_EINVAL instead of faulting the device.
#include "moe_kernels.h"

#define CHECK(cond)            \
  do {                         \
    if (!(cond)) return MOE_EINVAL; \
  } while (0)

static inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline int64_t tiles_of(int64_t S) { return (S + MOE_ROUTE_TILE - 1) / MOE_ROUTE_TILE; }

extern "C" {

int moe_abi_version(void) { return MOE_ABI_VERSION; }

int moe_topk_gate(const void* logits, int dtype, int64_t S, int E, int k, int32_t* ids,
                  void* gate_probs, void* probs, void* stream) {
  CHECK(S >= 0 && E >= 1 && (k == 1 || k == 2) && k <= E);
  CHECK(dtype == MOE_F32 || dtype == MOE_F64);
  if (S == 0) return MOE_OK;
  CHECK(logits && ids && gate_probs);
  return moe::launch_topk_gate(logits, dtype, S, E, k, ids, gate_probs, probs, S_(stream));
}

int moe_plan_tiles(const int32_t* ids, int64_t S, int E, int k, int32_t* local_rank,
                   int32_t* tile_counts, void* stream) {
  CHECK(S >= 0 && E >= 1 && E <= 3072 && (k == 1 || k == 2));
  if (S == 0) return MOE_OK;
  CHECK(ids && local_rank && tile_counts);
  return moe::launch_plan(ids, S, k, E, 0, nullptr, local_rank, tile_counts, nullptr, nullptr,
                          nullptr, nullptr, true, false, false, S_(stream));
}

int moe_plan_scan(const int32_t* tile_counts, int64_t S, int E, int64_t cap,
                  const int32_t* rank_base, int32_t* tile_offsets, int32_t* totals, int32_t* kept,
                  void* stream) {
  CHECK(S >= 0 && E >= 1 && cap >= 0);
  CHECK(totals && kept && (S == 0 || (tile_counts && tile_offsets)));
  return moe::launch_plan(nullptr, S, 1, E, cap, rank_base, nullptr,
                          const_cast<int32_t*>(tile_counts), tile_offsets, totals, kept, nullptr,
                          false, true, false, S_(stream));
}

int moe_plan_slots(const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                   int64_t S, int E, int k, int64_t cap, int32_t* slots, void* stream) {
  CHECK(S >= 0 && E >= 1 && (k == 1 || k == 2) && cap >= 0);
  if (S == 0) return MOE_OK;
  CHECK(ids && local_rank && tile_offsets && slots);
  return moe::launch_plan(ids, S, k, E, cap, nullptr, const_cast<int32_t*>(local_rank), nullptr,
                          const_cast<int32_t*>(tile_offsets), nullptr, nullptr, slots, false,
                          false, true, S_(stream));
}

size_t moe_plan_workspace_bytes(int64_t S, int E, int k) {
  if (S < 0 || E < 1 || k < 1) return 0;
  const int64_t T = tiles_of(S);
  return (size_t)(S * k + 2 * T * E + E) * sizeof(int32_t);
}

int moe_build_plan(const int32_t* ids, int64_t S, int E, int k, int64_t cap, int32_t* slots,
                   int32_t* expert_load, void* ws, size_t ws_bytes, void* stream) {
  CHECK(S >= 0 && E >= 1 && E <= 3072 && (k == 1 || k == 2) && cap >= 0 && expert_load);
  CHECK(ws_bytes >= moe_plan_workspace_bytes(S, E, k) && ws);
  const int64_t T = tiles_of(S);
  int32_t* w = static_cast<int32_t*>(ws);
  int32_t* local_rank = w;
  int32_t* tile_counts = local_rank + S * k;
  int32_t* tile_offsets = tile_counts + T * E;
  int32_t* totals = tile_offsets + T * E;
  if (S > 0) CHECK(ids && slots);
  return moe::launch_plan(ids, S, k, E, cap, nullptr, local_rank, tile_counts, tile_offsets, totals,
                          expert_load, slots, S > 0, true, S > 0, S_(stream));
}

size_t moe_scan_workspace_bytes(int64_t n) {
  if (n < 0) return 0;
  return (size_t)moe::scan_i64_workspace_elems(n) * sizeof(int64_t);
}

int moe_exclusive_scan_i64(const int64_t* in, int64_t n, int64_t* out, void* ws, size_t ws_bytes,
                           void* stream) {
  CHECK(n >= 0);
  if (n == 0) return MOE_OK;
  CHECK(in && out && ws && ws_bytes >= moe_scan_workspace_bytes(n));
  return moe::launch_scan_i64(in, n, out, static_cast<int64_t*>(ws), S_(stream));
}

int moe_blelloch_scan_f64(double* tree, int64_t m, void* stream) {
  CHECK(m >= 1 && (m & (m - 1)) == 0 && tree);
  return moe::launch_blelloch_f64(tree, m, S_(stream));
}

int moe_scatter(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                const int32_t* ids, const int32_t* slots, void* buf, uint8_t* occupied,
                void* stream) {
  CHECK(S >= 0 && row_bytes >= 0 && E >= 1 && (k == 1 || k == 2) && cap >= 0);
  CHECK(row_bytes % 2 == 0);
  if (S == 0 || cap == 0) return MOE_OK;
  CHECK(x && ids && slots && buf);
  moe::ScatterArgs a;
  a.x = static_cast<const uint8_t*>(x);
  a.S = S, a.row_bytes = row_bytes, a.k = k, a.E = E, a.cap = cap;
  a.ids = ids, a.slots = const_cast<int32_t*>(slots);
  a.buf = static_cast<uint8_t*>(buf), a.occupied = occupied;
  return moe::launch_scatter(a, S_(stream));
}

int moe_dispatch(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                 const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                 int32_t* slots, void* buf, void* stream) {
  CHECK(S >= 0 && row_bytes >= 0 && row_bytes % 2 == 0 && E >= 1 && (k == 1 || k == 2) &&
        cap >= 0);
  if (S == 0) return MOE_OK;
  CHECK(x && ids && local_rank && tile_offsets && slots && (buf || cap == 0));
  moe::ScatterArgs a;
  a.x = static_cast<const uint8_t*>(x);
  a.S = S, a.row_bytes = row_bytes, a.k = k, a.E = E, a.cap = cap;
  a.ids = ids, a.slots = slots, a.local_rank = local_rank, a.tile_offsets = tile_offsets;
  a.buf = static_cast<uint8_t*>(buf);
  return moe::launch_scatter(a, S_(stream));
}

int moe_dispatch_fused(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                       const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                       const float* gate_probs, int32_t* slots, void* buf, int32_t* row_token,
                       float* row_prob, void* out_dropped, void* stream) {
  CHECK(S >= 0 && row_bytes >= 0 && row_bytes % 2 == 0 && E >= 1 && (k == 1 || k == 2) &&
        cap >= 0);
  if (S == 0) return MOE_OK;
  // buf == NULL: route only (slots, row_token/row_prob, out = x for dropped tokens);
  // the GEMM then gathers the rows from x (moe_grouped_gemm_bf16_gather)
  CHECK(x && ids && local_rank && tile_offsets && gate_probs && slots && row_token && row_prob);
  moe::ScatterArgs a;
  a.x = static_cast<const uint8_t*>(x);
  a.S = S, a.row_bytes = row_bytes, a.k = k, a.E = E, a.cap = cap;
  a.ids = ids, a.slots = slots, a.local_rank = local_rank, a.tile_offsets = tile_offsets;
  a.buf = static_cast<uint8_t*>(buf);
  a.gate_probs = gate_probs, a.row_token = row_token, a.row_prob = row_prob;
  a.out_dropped = static_cast<uint8_t*>(out_dropped);
  return moe::launch_scatter(a, S_(stream));
}

int moe_dispatch_ep(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                    const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                    const int32_t* slot_base, const int32_t* row_base, int32_t* slots,
                    int32_t* row_index, void* send_buf, void* stream) {
  CHECK(S >= 0 && row_bytes >= 0 && row_bytes % 2 == 0 && E >= 1 && (k == 1 || k == 2) &&
        cap >= 0);
  if (S == 0) return MOE_OK;
  CHECK(x && ids && local_rank && tile_offsets && slot_base && row_base && slots && row_index);
  moe::ScatterArgs a;
  a.x = static_cast<const uint8_t*>(x);
  a.S = S, a.row_bytes = row_bytes, a.k = k, a.E = E, a.cap = cap;
  a.ids = ids, a.slots = slots, a.local_rank = local_rank, a.tile_offsets = tile_offsets;
  a.buf = static_cast<uint8_t*>(send_buf);
  a.slot_base = slot_base, a.row_base = row_base, a.row_index = row_index;
  return moe::launch_scatter(a, S_(stream));
}

int moe_combine(const void* y, int dtype, int64_t S, int M, int E, int k, int64_t cap,
                const int32_t* ids, const int32_t* slots, const int32_t* row_index,
                const void* gate_probs, int gp_dtype, const void* x_resid, const void* shared_out,
                void* out, int expert_order, void* stream) {
  CHECK(S >= 0 && M >= 0 && E >= 1 && (k == 1 || k == 2) && cap >= 0);
  if (S == 0 || M == 0) return MOE_OK;
  CHECK(ids && gate_probs && out && (row_index || slots));
  CHECK(y || cap == 0 || row_index);
  return moe::launch_combine(y, dtype, S, M, k, E, cap, ids, slots, row_index, gate_probs, gp_dtype,
                             x_resid, shared_out, out, expert_order, S_(stream));
}

int moe_gate_gemm_bf16(const void* x, const void* wg_t, int64_t S, int M, int E, int k,
                       float* logits, int32_t* ids, float* gate_probs, int32_t* local_rank,
                       int32_t* tile_counts, void* stream) {
  CHECK(S >= 0 && M >= 8 && M % 8 == 0 && E >= 1 && E <= 256 && (k == 1 || k == 2) && k <= E);
  if (S == 0) return MOE_OK;
  CHECK(x && wg_t && ids && gate_probs && local_rank && tile_counts);
  return moe::launch_gate_gemm_bf16(x, wg_t, S, M, E, k, logits, ids, gate_probs, local_rank,
                                    tile_counts, S_(stream));
}

int moe_gate_gemm_bf16_stats(const void* x, const void* wg_t, int64_t S, int M, int E, int k,
                             float* logits, int32_t* ids, float* gate_probs, int32_t* local_rank,
                             int32_t* tile_counts, float* probsum, void* stream) {
  CHECK(S >= 0 && M >= 8 && M % 8 == 0 && E >= 1 && E <= 256 && (k == 1 || k == 2) && k <= E);
  if (S == 0) return MOE_OK;
  CHECK(x && wg_t && ids && gate_probs && local_rank && tile_counts && probsum);
  return moe::launch_gate_gemm_bf16(x, wg_t, S, M, E, k, logits, ids, gate_probs, local_rank,
                                    tile_counts, S_(stream), probsum);
}

size_t moe_load_balance_workspace_bytes(int E) { return E < 1 ? 0 : 2 * (size_t)E * sizeof(double); }

int moe_load_balance_loss(const int32_t* ids, int64_t S, int E, int k, const void* probs, int dtype,
                          double* out, void* ws, size_t ws_bytes, void* stream) {
  CHECK(S >= 0 && E >= 1 && (k == 1 || k == 2) && out && ws);
  CHECK(ws_bytes >= moe_load_balance_workspace_bytes(E));
  CHECK(dtype == MOE_F32 || dtype == MOE_F64);
  if (S > 0) CHECK(ids && probs);
  return moe::launch_aux_loss(ids, S, k, E, probs, dtype, nullptr, nullptr, out,
                              static_cast<double*>(ws), S_(stream));
}

int moe_load_balance_loss_from_stats(const int32_t* counts, const float* probsum, int64_t S, int E,
                                     int k, double* out, void* stream) {
  CHECK(S >= 0 && E >= 1 && (k == 1 || k == 2) && counts && probsum && out);
  return moe::launch_aux_loss(nullptr, S, k, E, nullptr, MOE_F32, counts, probsum, out, nullptr,
                              S_(stream));
}

int moe_grouped_gemm_bf16(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                          int N, const float* bias, void* D, int num_groups,
                          const int32_t* row_start, int64_t row_stride, const int32_t* rows,
                          int64_t rows_const, const int32_t* weight_idx, int64_t max_group_rows,
                          int act, void* stream) {
  CHECK(a_rows >= 0 && K >= 8 && K % 8 == 0 && N >= 1 && b_rows >= N && num_groups >= 1);
  // (bit 1 of pad_scratch carries MOE_GEMM_TILE256 to the launcher)
  const int pad_scratch = ((act & MOE_GEMM_PAD_SCRATCH) ? 1 : 0) | ((act & MOE_GEMM_TILE256) ? 2 : 0);
  act &= ~(MOE_GEMM_PAD_SCRATCH | MOE_GEMM_TILE256);
  CHECK(act == MOE_ACT_NONE || act == MOE_ACT_GELU);
  CHECK(max_group_rows >= 0 && rows_const >= 0);
  if (a_rows == 0 || max_group_rows == 0) return MOE_OK;
  CHECK(A && B && D);
  return moe::launch_grouped_gemm_bf16(A, a_rows, K, B, b_rows, N, bias, D, num_groups, row_start,
                                       row_stride, rows, rows_const, weight_idx, max_group_rows,
                                       act, S_(stream), nullptr, nullptr, nullptr, nullptr, 0,
                                       pad_scratch);
}

int moe_grouped_gemm_bf16_gather(const void* X, int64_t x_rows, const int32_t* row_index, int K,
                                 const void* B, int64_t b_rows, int N, const float* bias, void* D,
                                 int num_groups, int64_t row_stride, const int32_t* rows,
                                 int64_t rows_const, int64_t max_group_rows, int act,
                                 void* stream) {
  CHECK(x_rows >= 0 && K >= 8 && K % 8 == 0 && N >= 1 && b_rows >= N && num_groups >= 1 &&
        row_stride >= 1);
  const int pad_scratch = (act & MOE_GEMM_PAD_SCRATCH) ? 1 : 0;
  act &= ~MOE_GEMM_PAD_SCRATCH;
  CHECK(act == MOE_ACT_NONE || act == MOE_ACT_GELU);
  CHECK(max_group_rows >= 0 && max_group_rows <= row_stride && rows_const >= 0);
  if (x_rows == 0 || max_group_rows == 0) return MOE_OK;
  CHECK(X && row_index && B && D);
  return moe::launch_grouped_gemm_bf16(X, x_rows, K, B, b_rows, N, bias, D, num_groups, nullptr,
                                       row_stride, rows, rows_const, nullptr, max_group_rows, act,
                                       S_(stream), nullptr, nullptr, nullptr, nullptr, 0,
                                       pad_scratch, row_index);
}

int moe_grouped_gemm_bf16_combine(const void* A, int64_t a_rows, int K, const void* B,
                                  int64_t b_rows, int N, const float* bias, int num_groups,
                                  const int32_t* row_start, int64_t row_stride,
                                  const int32_t* rows, int64_t rows_const,
                                  const int32_t* weight_idx, int64_t max_group_rows,
                                  const int32_t* row_token, const float* row_prob,
                                  const void* x_resid, void* out, void* y_out, void* stream) {
  CHECK(a_rows >= 0 && K >= 8 && K % 8 == 0 && N >= 1 && b_rows >= N && num_groups >= 1);
  CHECK(max_group_rows >= 0 && rows_const >= 0);
  if (a_rows == 0 || max_group_rows == 0) return MOE_OK;
  CHECK(A && B && row_token && row_prob && x_resid && out);
  return moe::launch_grouped_gemm_bf16(A, a_rows, K, B, b_rows, N, bias, y_out, num_groups,
                                       row_start, row_stride, rows, rows_const, weight_idx,
                                       max_group_rows, 2, S_(stream), row_token, row_prob,
                                       x_resid, out);
}

int moe_residual_gemm_bf16(const void* A, int64_t a_rows, const void* A2, int64_t a2_rows,
                           int a2_group, int K, const void* B, int64_t b_rows, int N,
                           const float* bias, void* D, int num_groups, int64_t row_stride,
                           const int32_t* rows, const int32_t* weight_idx, int64_t max_group_rows,
                           int mode, int rc_group, const int32_t* ids, const int32_t* slots,
                           const float* gate_probs, int k, int64_t cap, const void* x, void* out,
                           int64_t S, const int32_t* row_index, void* stream) {
  CHECK(a_rows >= 0 && K >= 8 && K % 8 == 0 && N >= 8 && N % 8 == 0 && num_groups >= 1);
  CHECK(row_stride >= 1 && max_group_rows >= 0 && max_group_rows <= row_stride);
  CHECK(mode == 0 || mode == 1);
  CHECK(b_rows >= N);
  if (a_rows == 0 || max_group_rows == 0) return MOE_OK;
  CHECK(A && B && D && rows && weight_idx);
  if (mode == 1) {
    CHECK(A2 && a2_rows >= 0 && a2_group >= 0 && a2_group <= num_groups);
  } else {
    CHECK(rc_group >= 0 && rc_group <= num_groups && ids && (slots || row_index) && gate_probs &&
          x && out);
    CHECK(k == 1 || k == 2);
    CHECK(cap >= 0 && S >= 0);
  }
  return moe::launch_residual_gemm_bf16(A, a_rows, A2, a2_rows, a2_group, K, B, b_rows, N, bias, D,
                                        num_groups, row_stride, rows, weight_idx, max_group_rows,
                                        mode, rc_group, ids, slots, gate_probs, k, cap, x, out, S,
                                        S_(stream), row_index);
}

int moe_grouped_gemm_f32(const float* A, int K, const float* B, int N, const float* bias, float* D,
                         int num_groups, const int32_t* row_start, int64_t row_stride,
                         const int32_t* rows, int64_t rows_const, const int32_t* weight_idx,
                         int64_t max_group_rows, int act, void* stream) {
  CHECK(K >= 1 && N >= 1 && num_groups >= 1 && max_group_rows >= 0);
  CHECK(act == MOE_ACT_NONE || act == MOE_ACT_GELU);
  if (max_group_rows == 0) return MOE_OK;
  CHECK(A && B && D);
  return moe::launch_grouped_gemm_f32(A, K, B, N, bias, D, num_groups, row_start, row_stride, rows,
                                      rows_const, weight_idx, max_group_rows, act, S_(stream));
}

}  // extern "C"
