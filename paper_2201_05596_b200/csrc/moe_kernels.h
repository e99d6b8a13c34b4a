// Internal launcher prototypes (namespace moe), called by abi.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/moe_b200.h"

namespace moe {

int launch_topk_gate(const void* logits, int dtype, int64_t S, int E, int k, int32_t* ids,
                     void* gate_probs, void* probs, cudaStream_t st);

int launch_plan(const int32_t* ids, int64_t S, int k, int E, int64_t cap, const int32_t* base,
                int32_t* local_rank, int32_t* tile_counts, int32_t* tile_offsets, int32_t* totals,
                int32_t* kept, int32_t* slots, bool tiles, bool scan, bool do_slots,
                cudaStream_t st);

int64_t scan_i64_workspace_elems(int64_t n);
int launch_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* ws, cudaStream_t st);
int launch_blelloch_f64(double* tree, int64_t m, cudaStream_t st);

int launch_scatter(const void* x, int64_t S, int64_t row_bytes, int k, int E, int64_t cap,
                   const int32_t* ids, int32_t* slots, const int32_t* local_rank,
                   const int32_t* tile_offsets, void* buf, uint8_t* occupied,
                   const int32_t* slot_base, const int32_t* row_base, int32_t* row_index,
                   cudaStream_t st);

int launch_combine(const void* y, int dtype, int64_t S, int M, int k, int E, int64_t cap,
                   const int32_t* ids, const int32_t* slots, const int32_t* row_index,
                   const void* gate_probs, int gp_dtype, const void* x, const void* shared,
                   void* out, int expert_order, cudaStream_t st);

int launch_grouped_gemm_bf16(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                             int N, const float* bias, void* D, int G, const int32_t* row_start,
                             int64_t row_stride, const int32_t* rows, int64_t rows_const,
                             const int32_t* weight_idx, int64_t max_group_rows, int act,
                             cudaStream_t st);

int launch_gate_gemm_bf16(const void* x, const void* wg_t, int64_t S, int M, int E, int k,
                          float* logits, int32_t* ids, float* gate_probs, int32_t* local_rank,
                          int32_t* tile_counts, cudaStream_t st);

int launch_grouped_gemm_f32(const float* A, int K, const float* B, int N, const float* bias,
                            float* D, int G, const int32_t* row_start, int64_t row_stride,
                            const int32_t* rows, int64_t rows_const, const int32_t* weight_idx,
                            int64_t max_group_rows, int act, cudaStream_t st);

}  // namespace moe
