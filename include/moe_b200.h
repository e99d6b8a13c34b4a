/*
 * moe_b200.h - C ABI of the B200-native (sm_100a) MoE-layer forward path.
 *
 * Drop-in boundary for the reference package `moekit` (arXiv 2201.05596,
 * /root/reference/pkg). The reference is pure Python/NumPy and has no FFI of
 * its own: its boundary is the Python API of moekit.gating (gating.py:36-50)
 * and the layer half of moekit.arch (arch.py:45-63). Each entry point below
 * replaces the NumPy body of one of those functions (cited per function); the
 * Python package paper_2201_05596_b200 binds them with ctypes and keeps the
 * reference's names, argument meaning and exceptions.
 *
 * Conventions
 *  - All pointers are DEVICE pointers on the current CUDA device, allocated
 *    by the caller (the library does not allocate caller data). `stream` is a
 *    cudaStream_t passed as void*; every call is stream-ordered and
 *    asynchronous. Results depend only on the arguments (SPEC.md:198-199
 *    "pure"). The library does keep process-wide launch caches, all keyed by
 *    device ordinal and thread-safe: per-(kernel, device) dynamic-smem
 *    attributes, SM counts and resident-cluster counts, a per-device pool of
 *    device-side tile counters (dynamic GEMM scheduling) and a per-device side
 *    stream; plus the cuTensorMapEncodeTiled entry point and the MOE_* tuning
 *    environment variables, read once. One process may drive several GPUs
 *    from several threads.
 *  - Exception: moe_malloc-style helpers (moe_ipc_malloc/free, for peer-memory
 *    regions) allocate, because a cudaIpc handle needs its own allocation.
 *  - Routing tables are int32 on device: ids/slots/local_rank are (S, k)
 *    row-major, token-major flattening (gating.py:226). DROPPED slot = -1.
 *  - Return value: 0 on success, MOE_EINVAL for bad arguments (checked before
 *    any launch), MOE_ENODRV / MOE_ETMA for driver/tensor-map failures, or a
 *    positive cudaError_t from the launch.
 */
#ifndef MOE_B200_H_
#define MOE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_ABI_VERSION 1
#define MOE_OK 0
#define MOE_EINVAL (-22)
#define MOE_ENODRV (-1001)
#define MOE_ETMA (-1002)

#define MOE_ROUTE_TILE 128 /* tokens per routing tile */

enum { MOE_F32 = 0, MOE_BF16 = 1, MOE_F64 = 2 };
enum { MOE_ACT_NONE = 0, MOE_ACT_GELU = 1, MOE_ACT_GELU_SAVE = 3, MOE_ACT_GELU_BWD = 4 };

int moe_abi_version(void);

/* gating.top_k_gate (gating.py:142-163). logits (S, E) f32|f64; outputs
 * ids (S, k) in descending-logit order with ties to the lower index,
 * gate_probs (S, k) and optional probs (S, E) of the input dtype: the max-
 * shifted softmax over all E, NOT renormalised over the k choices. */
int moe_topk_gate(const void* logits, int dtype, int64_t S, int E, int k, int32_t* ids,
                  void* gate_probs, void* probs, void* stream);

/* gating.build_dispatch_plan (gating.py:211-247), split in three launches.
 * T = ceil(S / MOE_ROUTE_TILE).
 *  tiles: local_rank (S, k) = earlier same-expert assignments inside the
 *         token's tile; tile_counts (T, E).
 *  scan : tile_offsets (T, E) = rank_base[e] (nullable; the EP prefix over
 *         lower ranks) + exclusive scan over tiles; totals (E) = this batch's
 *         assignments per expert; kept (E) = how many of them fall below cap.
 *  slots: slots (S, k) = tile_offsets + local_rank, or -1 at/over cap. */
int moe_plan_tiles(const int32_t* ids, int64_t S, int E, int k, int32_t* local_rank,
                   int32_t* tile_counts, void* stream);
int moe_plan_scan(const int32_t* tile_counts, int64_t S, int E, int64_t cap,
                  const int32_t* rank_base, int32_t* tile_offsets, int32_t* totals,
                  int32_t* kept, void* stream);
int moe_plan_slots(const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                   int64_t S, int E, int k, int64_t cap, int32_t* slots, void* stream);

/* One-call plan: workspace = local_rank (S*k) | tile_counts (T*E) |
 * tile_offsets (T*E) | totals (E), all int32. expert_load = kept. */
size_t moe_plan_workspace_bytes(int64_t S, int E, int k);
int moe_build_plan(const int32_t* ids, int64_t S, int E, int k, int64_t cap, int32_t* slots,
                   int32_t* expert_load, void* ws, size_t ws_bytes, void* stream);

/* gating.exclusive_scan_blelloch (gating.py:171-203). Integer input: exact
 * int64 exclusive scan. Float input: the up-sweep/down-sweep over the zero-
 * padded power-of-two buffer `tree` (m elements, in place), so results
 * match the reference's float64 tree order bit for bit. */
size_t moe_scan_workspace_bytes(int64_t n);
int moe_exclusive_scan_i64(const int64_t* in, int64_t n, int64_t* out, void* ws, size_t ws_bytes,
                           void* stream);
int moe_blelloch_scan_f64(double* tree, int64_t m, void* stream);

/* gating.scatter_tokens (gating.py:255-278): buf[(e*cap + slot)] = x[t] for
 * kept assignments; rows are row_bytes wide (any dtype, exact copies).
 * occupied (E*cap bytes, nullable) gets 1 at filled slots. The caller zero-
 * fills buf/occupied first when it needs the reference's zero rows. */
int moe_scatter(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                const int32_t* ids, const int32_t* slots, void* buf, uint8_t* occupied,
                void* stream);

/* Layer-path dispatch: plan_slots fused into scatter (slots written out). */
int moe_dispatch(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                 const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                 int32_t* slots, void* buf, void* stream);

/* moe_dispatch plus, for the fused-combine path (k=1): row_token / row_prob
 * (E*cap, the token and gate probability behind each expert-buffer row) and,
 * when out_dropped is given, out_dropped[t] = x[t] for fully dropped tokens.
 * buf may be NULL (route only: no row copies; see moe_grouped_gemm_bf16_gather). */
int moe_dispatch_fused(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                       const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                       const float* gate_probs, int32_t* slots, void* buf, int32_t* row_token,
                       float* row_prob, void* out_dropped, void* stream);

/* Expert-parallel dispatch into the all-to-all send buffer. tile_offsets come
 * from moe_plan_scan with rank_base = slot_base (global slots); a kept
 * assignment (slot < cap) goes to send row row_base[e] + slot - slot_base[e]
 * (rows grouped by owner rank, then expert, then slot); row_index (S, k)
 * receives that row or -1, for the combine after the return all-to-all. */
int moe_dispatch_ep(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                    const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                    const int32_t* slot_base, const int32_t* row_base, int32_t* slots,
                    int32_t* row_index, void* send_buf, void* stream);

/* gating.combine_tokens (gating.py:281-307) and the combine + residual of
 * arch.forward_layer (arch.py:389-391, :395-413):
 *   out[t] = ((x_resid[t]) + sum_j gate_prob[t,j] * y[row(t,j)]) + shared_out[t]
 * row(t,j) = row_index[t,j] if row_index else ids*cap + slots (-1 = dropped).
 * expert_order=1 sums contributions in ascending expert id (forward_layer),
 * 0 in choice order (combine_tokens). dtype: F64 (gp F64, bit-exact adds),
 * F32 (gp F32) or BF16 (gp F32, fp32 accumulation). */
int moe_combine(const void* y, int dtype, int64_t S, int M, int E, int k, int64_t cap,
                const int32_t* ids, const int32_t* slots, const int32_t* row_index,
                const void* gate_probs, int gp_dtype, const void* x_resid, const void* shared_out,
                void* out, int expert_order, void* stream);

/* Gate GEMM (arch.py:384) fused with top_k_gate and plan_tiles on tcgen05:
 * x bf16 (S, M); wg_t bf16 (Epad, M) = gate_w^T zero-padded to Epad rows,
 * Epad = max(32, next_pow2(E)) <= 256. logits (S, E) f32 is optional. */
int moe_gate_gemm_bf16(const void* x, const void* wg_t, int64_t S, int M, int E, int k,
                       float* logits, int32_t* ids, float* gate_probs, int32_t* local_rank,
                       int32_t* tile_counts, void* stream);

/* As moe_gate_gemm_bf16, plus probsum (E) f32 += column sums of the full
 * softmax over the batch (caller zero-fills): with the plan scan's pre-drop
 * totals this gives the load-balance loss without re-reading anything. */
int moe_gate_gemm_bf16_stats(const void* x, const void* wg_t, int64_t S, int M, int E, int k,
                             float* logits, int32_t* ids, float* gate_probs, int32_t* local_rank,
                             int32_t* tile_counts, float* probsum, void* stream);

/* arch.load_balance_loss (arch.py:297-313): E * sum_e f_e * P_e with pre-drop
 * assignment fractions f_e = count_e / (S k) and P_e = mean_t probs[t, e],
 * written as one float64 to *out. From ids (S, k) + probs (S, E) f32|f64 with
 * a 2E-double workspace, or from the fused gate's statistics (counts = the
 * plan scan's totals, probsum from moe_gate_gemm_bf16_stats). */
size_t moe_load_balance_workspace_bytes(int E);
int moe_load_balance_loss(const int32_t* ids, int64_t S, int E, int k, const void* probs, int dtype,
                          double* out, void* ws, size_t ws_bytes, void* stream);
int moe_load_balance_loss_from_stats(const int32_t* counts, const float* probsum, int64_t S, int E,
                                     int k, double* out, void* stream);

/* Grouped expert GEMM on tcgen05 (the two halves of forward_ffn,
 * arch.py:368-369): for each group g with rows[g] rows starting at row
 * row_start[g] (or g*row_stride when row_start is NULL) of A (a_rows, K):
 *   D[rows] = act(A[rows] @ B_w^T + bias_w),  w = weight_idx[g] (or g)
 * A bf16 (a_rows, K); B bf16 (b_rows, K) with weight w at rows [w*N, w*N+N)
 * (i.e. W^T, K-major); bias f32 (nweights, N) nullable; D bf16 (a_rows, N).
 * rows == NULL means every group has rows_const rows. max_group_rows bounds
 * rows[g] (sizes the launch). act: MOE_ACT_NONE | MOE_ACT_GELU (tanh form),
 * optionally | MOE_GEMM_PAD_SCRATCH: the rows [rows[g], row_stride) of each
 * group's D block are scratch the kernel may overwrite (row_start == NULL), so
 * whole 32-row boxes go out through TMA tensor stores (the expert buffers'
 * padding rows; without the flag D rows past rows[g] are never written). */
#define MOE_GEMM_PAD_SCRATCH 0x100
/* act flag: keep 256-column tiles (no 256 x 512 tiles) - the expert-parallel owner
 * GEMM1, where the 512-column GELU tiles measured less even across ranks */
#define MOE_GEMM_TILE256 0x200
int moe_grouped_gemm_bf16(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                          int N, const float* bias, void* D, int num_groups,
                          const int32_t* row_start, int64_t row_stride, const int32_t* rows,
                          int64_t rows_const, const int32_t* weight_idx, int64_t max_group_rows,
                          int act, void* stream);

/* Grouped GEMM with A rows gathered by index (TMA tile::gather4): A row
 * (g*row_stride + r) = X[row_index[g*row_stride + r]] for r < rows[g]; D, bias,
 * B, act (incl. MOE_GEMM_PAD_SCRATCH) as moe_grouped_gemm_bf16 with row_start
 * NULL. The k=1 layer passes x and the row_token table of
 * moe_dispatch_fused(buf = NULL): the dispatch copy of scatter_tokens
 * (gating.py:255-278) is done by GEMM1's loads. */
int moe_grouped_gemm_bf16_gather(const void* X, int64_t x_rows, const int32_t* row_index, int K,
                                 const void* B, int64_t b_rows, int N, const float* bias, void* D,
                                 int num_groups, int64_t row_stride, const int32_t* rows,
                                 int64_t rows_const, int64_t max_group_rows, int act,
                                 void* stream);

/* Residual-MoE / PR-MoE layer (arch.py:389-391) with the shared MLP run as extra
 * groups of the expert launches. Groups are row_stride rows apart: groups
 * [0, E) are the experts (expert buffer rows, row_stride = capacity), groups
 * [E, G) the shared MLP over token blocks of row_stride rows (weight_idx E).
 *  mode 1 (GEMM1, bias + tanh-GELU, forward_ffn's first half arch.py:368-369):
 *    groups >= a2_group read their A rows from A2 (x) at row
 *    (g - a2_group) * row_stride + r instead of A (the dispatched buffer).
 *    D = (G * row_stride, N) bf16; rows past rows[g] are scratch.
 *  mode 0 (GEMM2): groups < rc_group store y = A @ B_w^T + bias_w to D (expert
 *    rows); groups >= rc_group (token t = (g - rc_group) * row_stride + r) emit
 *      out[t] = (x[t] + sum_j gate_probs[t, j] * y[ids[t, j] * cap + slots[t, j]])
 *               + (A[row] @ B_E^T + bias_E)
 *    over the kept choices in ascending expert order (forward_layer's order,
 *    arch.py:399-410), once every expert tile of the launch has stored its y.
 *  rows: (G) int32 device rows per group; weight_idx: (G) int32; bias (W, N).
 *  row_index (nullable, (S, k)): the y row of each choice (-1 = dropped) instead
 *    of ids * cap + slots - the expert-parallel source side, whose expert rows
 *    came back over NVLink into a (S * k)-row return buffer passed as D with
 *    rc_group = 0. */
int moe_residual_gemm_bf16(const void* A, int64_t a_rows, const void* A2, int64_t a2_rows,
                           int a2_group, int K, const void* B, int64_t b_rows, int N,
                           const float* bias, void* D, int num_groups, int64_t row_stride,
                           const int32_t* rows, const int32_t* weight_idx, int64_t max_group_rows,
                           int mode, int rc_group, const int32_t* ids, const int32_t* slots,
                           const float* gate_probs, int k, int64_t cap, const void* x, void* out,
                           int64_t S, const int32_t* row_index, void* stream);

/* GEMM2 of a k=1 layer with combine_tokens and the residual add fused into the
 * epilogue (gating.py:281-307, arch.py:389): for every expert-buffer row r
 *   out[row_token[r]] = x_resid[row_token[r]] + row_prob[r] * (A[r] @ B_w^T + bias_w)
 * row_token / row_prob come from moe_dispatch_fused, which also writes
 * out[t] = x[t] for fully dropped tokens. y_out (nullable, (a_rows, N) bf16)
 * additionally keeps the expert outputs A[r] @ B_w^T + bias_w per row (the
 * training forward needs them for the gate-probability gradient). Other
 * arguments as above. */
int moe_grouped_gemm_bf16_combine(const void* A, int64_t a_rows, int K, const void* B,
                                  int64_t b_rows, int N, const float* bias, int num_groups,
                                  const int32_t* row_start, int64_t row_stride,
                                  const int32_t* rows, int64_t rows_const,
                                  const int32_t* weight_idx, int64_t max_group_rows,
                                  const int32_t* row_token, const float* row_prob,
                                  const void* x_resid, void* out, void* y_out, void* stream);

/* fp32 SIMT variant (parity path). B f32 in the reference layout: weight w is
 * (K, N) row-major at B + w*K*N. */
int moe_grouped_gemm_f32(const float* A, int K, const float* B, int N, const float* bias, float* D,
                         int num_groups, const int32_t* row_start, int64_t row_stride,
                         const int32_t* rows, int64_t rows_const, const int32_t* weight_idx,
                         int64_t max_group_rows, int act, void* stream);

/* ---------------------------------------------------------------------------
 * Backward of the layer (training; the reference forward is tape-aware,
 * arch.py:375-377: gradients flow through the gate probabilities that scale
 * each expert's contribution, not through the routing decisions). bf16.
 * ------------------------------------------------------------------------- */

/* Training variants of the grouped GEMM: act = MOE_ACT_GELU_SAVE stores the
 * pre-activation a = A@B^T + bias into aux (same shape as D) and D = gelu(a);
 * act = MOE_ACT_GELU_BWD computes D = (A@B^T) * gelu'(aux) (aux = a). */
int moe_grouped_gemm_bf16_aux(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                              int N, const float* bias, void* D, int num_groups,
                              const int32_t* row_start, int64_t row_stride, const int32_t* rows,
                              int64_t rows_const, const int32_t* weight_idx,
                              int64_t max_group_rows, int act, void* aux, void* stream);

/* Through the combine (mul + take_elems vjps): for each kept (t, j) with
 * expert-buffer row r = ids*cap + slot: dy[r] = gate_prob * dout[t] (bf16)
 * and dp[t, j] = <dout[t], y[r]> (f32, 0 for dropped). */
int moe_combine_bwd_bf16(const void* dout, const void* y, int64_t S, int M, int E, int k,
                         int64_t cap, const int32_t* ids, const int32_t* slots,
                         const float* gate_probs, void* dy, float* dp, void* stream);

/* Through the gate softmax (row_softmax vjp, tensor.py:263-266):
 * dlogits[t] = s_t * (g_t - <g_t, s_t>) with s = softmax(logits[t]) and g
 * nonzero only at the kept choices (g[ids[t,j]] = dp[t,j]); bf16 (S, Epad), or
 * with split = 1 bf16 (S, 2*Epad) rows [hi | lo], hi + lo = dlogits to ~2^-16. */
int moe_gate_bwd(const float* logits, int64_t S, int E, int Epad, int k, const int32_t* ids,
                 const int32_t* slots, const float* dp, void* dlogits, int split, void* stream);

/* Bias gradients: out[g][c] += sum_{r < rows[g]} X[g*row_stride + r][c] (fp32;
 * caller zero-fills out (num_groups, W)); X bf16 row-major width W (W % 8 == 0). */
int moe_colsum_rows_bf16(const void* X, int W, int num_groups, int64_t row_stride,
                         const int32_t* rows, int64_t rows_const, float* out, void* stream);

/* Weight gradients straight from row-major activations (tcgen05, MN-major
 * operands, no transposes): D[g] (P x Q, bf16) = X_g^T Y_g where X_g, Y_g are
 * rows [g*k_stride, g*k_stride + k_rows[g]) of X (x_rows x P) and Y (x_rows x Q);
 * k_rows nullable -> k_rows_const; groups with no rows get zeros. Rows past
 * k_rows[g] are never used (may hold anything). P, Q multiples of 8. */
int moe_grouped_gemm_bf16_wgrad(const void* X, int64_t x_rows, int P, const void* Y, int Q,
                                int num_groups, int64_t k_stride, const int32_t* k_rows,
                                int64_t k_rows_const, void* D, void* stream);

/* D (P x Q, fp32) += X^T Y over all `rows` (split-K across the SMs, fp32
 * reduction; caller zero-fills D): gate and shared-MLP weight gradients. */
int moe_gemm_bf16_wgrad_f32(const void* X, int64_t rows, int P, const void* Y, int Q, float* D,
                            void* stream);

/* dx[t] = dout[t] + sum_j kept dxr[ids*cap + slot] + extra1[t] (+ extra2[t]); M % 8 == 0. */
int moe_bwd_dx_bf16(const void* dout, const void* dxr, int64_t S, int M, int E, int k, int64_t cap,
                    const int32_t* ids, const int32_t* slots, const void* extra1,
                    const void* extra2, void* dx, void* stream);

/* ---------------------------------------------------------------------------
 * Expert parallelism over NVLink peer memory (one process per GPU of a box).
 * Replaces the two all-to-alls of the EP layer (new; placement after
 * planner.py:101-109, delivery order of commsim.py:188-189) with stores fused
 * into the dispatch kernel and the GEMM2 epilogue.
 * ------------------------------------------------------------------------- */

/* Device memory shareable with the other ranks' processes (cudaMalloc +
 * cudaIpc handles; 64-byte handles, exchanged by the caller). Zero-filled. */
/* Direct peer access from the current device to peer_device's memory (one
 * process driving several GPUs, e.g. tools/nvlink_ep_probe.py); 0 if enabled
 * or already enabled. */
int moe_enable_peer_access(int peer_device);

int moe_ipc_malloc(size_t bytes, void** ptr);
int moe_ipc_free(void* ptr);
int moe_ipc_get_handle(void* ptr, void* handle64);
int moe_ipc_open_handle(const void* handle64, void** ptr);
int moe_ipc_close_handle(void* ptr);

/* Global-capacity exchange plan on device from the all-gathered counts
 * (world, E) int32: slot_base (E) = assignments to e on lower ranks;
 * row_base (E) = first row of this rank's rows for e in the owner's receive
 * buffer, laid out [local expert][global slot] (sources in rank order, i.e.
 * the single-GPU expert buffer without padding); as an owner, seg_start /
 * seg_rows (E/world) per local expert and recv_rows (1). */
int moe_ep_plan(const int32_t* counts, int world, int rank, int E, int64_t cap, int32_t* slot_base,
                int32_t* row_base, int32_t* seg_start, int32_t* seg_rows, int32_t* recv_rows,
                void* stream);

/* moe_ep_plan with the padded receive layout: local expert j owns rows
 * [j*cap, (j+1)*cap), row = j*cap + global slot (the single-GPU expert buffer);
 * seg_start[j] = j*cap. The owner's grouped GEMMs then run with a uniform group
 * stride (row_start NULL, row_stride = cap). */
int moe_ep_plan_padded(const int32_t* counts, int world, int rank, int E, int64_t cap,
                       int32_t* slot_base, int32_t* row_base, int32_t* seg_start, int32_t* seg_rows,
                       int32_t* recv_rows, void* stream);

/* moe_ep_plan for C token chunks per rank (chunk c of rank s = its tokens
 * [c*S/C, (c+1)*S/C)): counts (world, C, E); outputs per chunk: slot_base
 * (C, E), row_base (C, E), seg_start / seg_rows (C, E/world), recv_rows (C);
 * the owners' receive buffers are chunk-major, so chunk c can be exchanged
 * while chunk c-1 is in the GEMMs. C = 1 is moe_ep_plan. */
int moe_ep_plan_chunked(const int32_t* counts, int world, int rank, int E, int chunks, int64_t cap,
                        int32_t* slot_base, int32_t* row_base, int32_t* seg_start,
                        int32_t* seg_rows, int32_t* recv_rows, void* stream);

/* Launch limits of the calling host thread (0 = none): the persistent GEMMs
 * use at most gemm_ctas CTAs and the dispatch / pull copy kernels at most
 * comm_blocks blocks, so an exchange can run beside a GEMM on the SMs left. */
int moe_set_launch_limits(int gemm_ctas, int comm_blocks);

/* System-scope flag barrier over peer signal pads: epoch = *epoch_counter + 1
 * (a device counter, so the barrier can be captured in a CUDA graph) is
 * written into slot [rank] of every peer's pad (peer_signal: device array of
 * world pointers); waits until my_signal[i] >= epoch for all i. Bounded: sets
 * *error_flag = 1 after ~10 s instead of hanging. */
int moe_ipc_barrier(int* const* peer_signal, int* my_signal, int world, int rank,
                    int* epoch_counter, int* error_flag, void* stream);

/* All-gather of n int32 per rank over peer memory fused with the barrier
 * above: src (n) goes to slot [rank] of every peer's (world, n) array
 * (peer_dst: device array of world pointers). Used for the per-expert counts
 * of the EP layer, so no NCCL call sits on its data path. */
int moe_ipc_allgather_i32(const int32_t* src, int n, int32_t* const* peer_dst, int world, int rank,
                          int* const* peer_signal, int* my_signal, int* epoch_counter,
                          int* error_flag, void* stream);

/* Dispatch straight into the owners' receive buffers over NVLink: kept row
 * (t, j) of expert e goes to peer_recv[e / e_per_rank] at row
 * row_base[e] + slot - slot_base[e], with its token index and gate
 * probability to peer_token / peer_prob (device arrays of world pointers);
 * row_index (S, k) gets that owner-side row (or -1). Fully dropped tokens:
 * out_dropped[t] = x[t] (local; nullable). peer_src (nullable; device array of
 * world int32 pointers) selects the push return: each receive row also records
 * its source (my_rank) and return row t*k + j (in peer_token), and row_index
 * gets the return row t*k + j instead of the owner-side row. */
int moe_dispatch_p2p(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                     const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                     const float* gate_probs, const int32_t* slot_base, const int32_t* row_base,
                     int e_per_rank, void* const* peer_recv, int32_t* const* peer_token,
                     float* const* peer_prob, int32_t* slots, int32_t* row_index,
                     void* out_dropped, int32_t* const* peer_src, int my_rank, void* stream);

/* Owner side of the push return (any k, Residual-MoE included): GEMM2 over the
 * receive buffer, every valid row r stored straight back over NVLink to rank
 * row_src[r]'s buffer push_base[row_src[r]] at row row_token[r]:
 *  combine = 1 (k = 1 layers): the combined row x_r + row_prob[r] * (acc + b2)
 *    (x_r = x_rows[r], the dispatched token row), into the source's output;
 *  combine = 0: y = acc + b2, into the source's (S * k)-row return buffer, which
 *    the source then combines locally (moe_combine / moe_residual_gemm_bf16).
 * row_token / row_src / row_prob come from moe_dispatch_p2p with peer_src set.
 * Groups start at row_start[g] or, with row_start NULL, at g * row_stride. */
int moe_grouped_gemm_bf16_push(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                               int N, const float* bias, int num_groups, const int32_t* row_start,
                               int64_t row_stride, const int32_t* rows, const int32_t* weight_idx,
                               int64_t max_group_rows, int combine, const int32_t* row_token,
                               const float* row_prob, const int32_t* row_src,
                               void* const* push_base, const void* x_rows, void* stream);

/* Owner side of a k=1 EP layer: GEMM2 + combine + residual, in the receive
 * layout: out_rows[r] = x_rows[r] + row_prob[r] * (A[r] @ B_w^T + b_w), with
 * x_rows = the dispatched token rows (GEMM1's input). */
int moe_grouped_gemm_bf16_combine_rows(const void* A, int64_t a_rows, int K, const void* B,
                                       int64_t b_rows, int N, const float* bias, int num_groups,
                                       const int32_t* row_start, const int32_t* rows,
                                       const int32_t* weight_idx, int64_t max_group_rows,
                                       const int32_t* row_token, const float* row_prob,
                                       const void* x_rows, void* out_rows, void* stream);

/* Row permutation dst[i] = src[index[i]] (i < n; row_bytes % 16 == 0): the
 * layout transforms of the hierarchical and coordinated all-to-all schedules
 * (commsim.py:280-464 "layout-transform" steps). */
int moe_gather_rows(const void* src, int64_t row_bytes, const int32_t* index, int64_t n,
                    void* dst, void* stream);

/* Source side (k=1): out[t] = peer_rows[owner(ids[t])][row_index[t]] over
 * NVLink for every kept token (peer_rows: device array of world pointers). */
int moe_pull_rows_p2p(int64_t S, int64_t row_bytes, int E, int k, const int32_t* ids,
                      const int32_t* row_index, int e_per_rank, void* const* peer_rows, void* out,
                      void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MOE_B200_H_ */
