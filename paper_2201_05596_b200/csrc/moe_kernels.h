// Internal launcher prototypes (namespace moe), called by abi.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/moe_b200.h"

namespace moe {

// MOE_PDL (default 0): launch the forward hot-path kernels with programmatic
// dependent launch (see pdl_wait / pdl_trigger in common.cuh)
bool pdl_on();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

int launch_topk_gate(const void* logits, int dtype, int64_t S, int E, int k, int32_t* ids,
                     void* gate_probs, void* probs, cudaStream_t st);

int launch_plan(const int32_t* ids, int64_t S, int k, int E, int64_t cap, const int32_t* base,
                int32_t* local_rank, int32_t* tile_counts, int32_t* tile_offsets, int32_t* totals,
                int32_t* kept, int32_t* slots, bool tiles, bool scan, bool do_slots,
                cudaStream_t st);

int64_t scan_i64_workspace_elems(int64_t n);
int launch_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* ws, cudaStream_t st);
int launch_blelloch_f64(double* tree, int64_t m, cudaStream_t st);

struct ScatterArgs {
  const uint8_t* x = nullptr;        // (S, row_bytes)
  int64_t S = 0, row_bytes = 0;
  int k = 1, E = 1;
  int64_t cap = 0;
  const int32_t* ids = nullptr;
  int32_t* slots = nullptr;               // read (API scatter) or written (layer dispatch)
  const int32_t* local_rank = nullptr;    // non-null: resolve slots from the plan tables
  const int32_t* tile_offsets = nullptr;
  uint8_t* buf = nullptr;
  uint8_t* occupied = nullptr;
  const int32_t* slot_base = nullptr;     // EP: rank prefix per expert
  const int32_t* row_base = nullptr;      // EP: send-buffer start row per expert
  int32_t* row_index = nullptr;           // EP: (S, k) send row or -1
  const float* gate_probs = nullptr;      // fused combine: (S, k)
  int32_t* row_token = nullptr;           // fused combine: per buffer row -> token
  float* row_prob = nullptr;              // fused combine: per buffer row -> gate prob
  uint8_t* out_dropped = nullptr;         // fused combine: out rows of fully dropped tokens
  // EP over NVLink peer memory: per-rank receive buffer / row_token / row_prob bases
  // (device arrays of `world` pointers); owner of expert e = e / e_per_rank
  uint8_t* const* peer_buf = nullptr;
  int32_t* const* peer_token = nullptr;
  float* const* peer_prob = nullptr;
  int e_per_rank = 1;
  // EP push return: the owner's GEMM2 epilogue stores each row straight back to its
  // source. Per receive row the owner gets the source rank (peer_src) and the
  // return row t*k + j (peer_token); row_index (S, k) becomes that return row
  // (or -1 when dropped)
  int32_t* const* peer_src = nullptr;
  int my_rank = 0;
};

int launch_scatter(const ScatterArgs& args, cudaStream_t st);

int launch_combine(const void* y, int dtype, int64_t S, int M, int k, int E, int64_t cap,
                   const int32_t* ids, const int32_t* slots, const int32_t* row_index,
                   const void* gate_probs, int gp_dtype, const void* x, const void* shared,
                   void* out, int expert_order, cudaStream_t st);

int launch_grouped_gemm_bf16(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                             int N, const float* bias, void* D, int G, const int32_t* row_start,
                             int64_t row_stride, const int32_t* rows, int64_t rows_const,
                             const int32_t* weight_idx, int64_t max_group_rows, int act,
                             cudaStream_t st, const int32_t* row_token = nullptr,
                             const float* row_prob = nullptr, const void* x_resid = nullptr,
                             void* out = nullptr, int x_by_row = 0, int pad_scratch = 0,
                             const int32_t* a_gather = nullptr, void* const* push_base = nullptr,
                             const int32_t* row_src = nullptr);

int launch_residual_gemm_bf16(const void* A, int64_t a_rows, const void* A2, int64_t a2_rows,
                              int a2_group, int K, const void* B, int64_t b_rows, int N,
                              const float* bias, void* D, int G, int64_t row_stride,
                              const int32_t* rows, const int32_t* weight_idx,
                              int64_t max_group_rows, int mode, int rc_group, const int32_t* ids,
                              const int32_t* slots, const float* gp, int k, int64_t cap,
                              const void* x, void* out, int64_t S, cudaStream_t st,
                              const int32_t* row_index = nullptr);

int launch_wgrad_bf16(const void* X, int64_t x_rows, int P, const void* Y, int Q, int G,
                      int64_t k_stride, const int32_t* k_rows, int64_t k_rows_const, void* D,
                      int acc, cudaStream_t st);

// expert parallelism over NVLink peer memory (ep_p2p.cu)
void set_launch_limits(int gemm_ctas, int comm_blocks);
int gemm_cta_limit();
int comm_block_limit();
int launch_ep_plan(const int32_t* counts, int world, int rank, int E, int C, int64_t cap,
                   int32_t* slot_base, int32_t* row_base, int32_t* seg_start, int32_t* seg_rows,
                   int32_t* recv_rows, cudaStream_t st, int padded = 0);
int launch_pull_rows(int64_t S, int64_t row_bytes, int k, int e_per_rank, const int32_t* ids,
                     const int32_t* row_index, uint8_t* const* peer_rows, uint8_t* out,
                     cudaStream_t st);
int launch_gather_rows(const uint8_t* src, int64_t row_bytes, const int32_t* index, int64_t n,
                       uint8_t* dst, cudaStream_t st);
int launch_ipc_allgather(const int32_t* src, int n, int32_t* const* peer_dst, int world, int rank,
                         int* const* peer_signal, int* my_signal, int* epoch_counter,
                         int* error_flag, cudaStream_t st);
int launch_ipc_barrier(int* const* peer_signal, int* my_signal, int world, int rank,
                       int* epoch_counter, int* error_flag, cudaStream_t st);

int launch_gate_gemm_bf16(const void* x, const void* wg_t, int64_t S, int M, int E, int k,
                          float* logits, int32_t* ids, float* gate_probs, int32_t* local_rank,
                          int32_t* tile_counts, cudaStream_t st, float* probsum = nullptr);

// load-balance loss (arch.py:297-313)
int launch_aux_loss(const int32_t* ids, int64_t S, int k, int E, const void* probs, int dtype,
                    const int32_t* counts, const float* probsum, double* out, double* ws,
                    cudaStream_t st);

int launch_grouped_gemm_f32(const float* A, int K, const float* B, int N, const float* bias,
                            float* D, int G, const int32_t* row_start, int64_t row_stride,
                            const int32_t* rows, int64_t rows_const, const int32_t* weight_idx,
                            int64_t max_group_rows, int act, cudaStream_t st);

}  // namespace moe
