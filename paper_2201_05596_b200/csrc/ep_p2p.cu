// Expert parallelism over NVLink peer memory (one process per GPU, one box).
//
//   * moe_ipc_*      : cudaMalloc'd regions shared between the ranks' processes
//                      (cudaIpc handles exchanged by the caller over NCCL)
//   * ep_plan_kernel : from the all-gathered (world, E) expert counts, the
//                      global-capacity exchange plan on device (no host sync):
//                      this rank's slot prefix per expert, where its rows land
//                      in each owner's receive buffer, and (as an owner) the
//                      per-local-expert row ranges of its own receive buffer
//   * ipc_barrier    : a system-scope release/acquire flag exchange between the
//                      ranks (bounded spin: sets an error flag after ~10 s
//                      instead of hanging)
// The data movement is fused into the kernels around the GEMMs: the dispatch
// kernel stores token rows straight into the owners' receive buffers; the owner's
// GEMM2 epilogue combines (x + p*y) in place in its receive layout, and the
// source pulls its rows back with wide NVLink loads (pull_rows_kernel).
#include "common.cuh"
#include "moe_kernels.h"

#include <string.h>

namespace moe {

// Launch limits for overlapping an exchange with the GEMMs on one GPU: the GEMM
// leaves SMs free (persistent grid capped) and the copy kernels stay inside
// them. Thread-local (set around the launches by the host thread issuing them).
static thread_local int t_gemm_ctas = 0, t_comm_blocks = 0;
void set_launch_limits(int gemm_ctas, int comm_blocks) {
  t_gemm_ctas = gemm_ctas;
  t_comm_blocks = comm_blocks;
}
int gemm_cta_limit() { return t_gemm_ctas; }
int comm_block_limit() { return t_comm_blocks; }

// Exchange plan from the all-gathered per-(rank, chunk, expert) counts, C >= 1
// token chunks per rank (chunk c of rank s = its tokens [c*S/C, (c+1)*S/C)).
// Global token order is (rank, chunk, token), so the global slot of my first
// chunk-c assignment to e is base = sum of the counts before (rank, c), and the
// kept rows are clamp(cap - base, 0, count).
// Owner o's receive buffer is chunk-major, each chunk expert-major:
//   [chunk c][local expert j][source s][rows in slot order]
// (C = 1: the single-GPU expert buffer without padding). Outputs per chunk c:
// slot_base[c][e], row_base[c][e] (my first chunk-c row for e in its owner's
// buffer), seg_start/seg_rows[c][j] (my buffer as an owner), recv_rows[c].
// padded (C = 1 only): every local expert owns cap rows, row = e_loc * cap + global
// slot - the single-GPU expert buffer's layout, so the owner's grouped GEMMs run
// with a uniform group stride (TMA-store epilogues, 256 x 512 tiles)
__global__ void ep_plan_kernel(const int32_t* __restrict__ counts, int world, int rank, int E,
                               int C, int64_t cap, int32_t* __restrict__ slot_base,
                               int32_t* __restrict__ row_base, int32_t* __restrict__ seg_start,
                               int32_t* __restrict__ seg_rows, int32_t* __restrict__ recv_rows,
                               int padded) {
  extern __shared__ int kept[];  // [world][C][E], then chunk_off [world][C]
  int* chunk_off = kept + world * C * E;
  const int e_loc = E / world;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int64_t base = 0;
    for (int s = 0; s < world; ++s)
      for (int c = 0; c < C; ++c) {
        const int cnt = counts[(s * C + c) * E + e];
        int64_t kp = cap - base;
        kp = kp < 0 ? 0 : (kp > cnt ? cnt : kp);
        kept[(s * C + c) * E + e] = (int)kp;
        if (s == rank) slot_base[c * E + e] = (int)base;
        base += cnt;
      }
  }
  __syncthreads();
  // chunk offsets of every owner's buffer
  for (int i = threadIdx.x; i < world; i += blockDim.x) {
    int64_t run = 0;
    for (int c = 0; c < C; ++c) {
      chunk_off[i * C + c] = (int)run;
      for (int j = 0; j < e_loc; ++j)
        for (int s = 0; s < world; ++s) run += kept[(s * C + c) * E + i * e_loc + j];
    }
  }
  __syncthreads();
  if (padded) {
    for (int e = threadIdx.x; e < E; e += blockDim.x)
      row_base[e] = (int)((e % e_loc) * cap + slot_base[e]);
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t tot = 0;
      for (int j = 0; j < e_loc; ++j) {
        int64_t r = 0;
        for (int s = 0; s < world; ++s) r += kept[s * E + rank * e_loc + j];
        seg_start[j] = (int)(j * cap);
        seg_rows[j] = (int)r;
        tot += r;
      }
      recv_rows[0] = (int)tot;
    }
    return;
  }
  for (int ce = threadIdx.x; ce < C * E; ce += blockDim.x) {
    const int c = ce / E, e = ce % E;
    const int o = e / e_loc, el = e % e_loc;
    int64_t st = chunk_off[o * C + c];
    for (int j = 0; j < el; ++j)
      for (int s = 0; s < world; ++s) st += kept[(s * C + c) * E + o * e_loc + j];
    for (int s = 0; s < rank; ++s) st += kept[(s * C + c) * E + e];
    row_base[c * E + e] = (int)st;
  }
  for (int c = threadIdx.x; c < C; c += blockDim.x) {  // as an owner: one group per local expert
    int64_t run = chunk_off[rank * C + c];
    const int64_t start = run;
    for (int j = 0; j < e_loc; ++j) {
      int64_t r = 0;
      for (int s = 0; s < world; ++s) r += kept[(s * C + c) * E + rank * e_loc + j];
      seg_start[c * e_loc + j] = (int)run;
      seg_rows[c * e_loc + j] = (int)r;
      run += r;
    }
    recv_rows[c] = (int)(run - start);
  }
}

// The epoch lives in device memory (incremented here), so the barrier is
// CUDA-graph safe: a replayed graph keeps advancing it.
__global__ void ipc_barrier_kernel(int* const* __restrict__ peer_signal, int* my_signal, int world,
                                   int rank, int* epoch_counter, int* error_flag) {
  __shared__ int epoch_s;
  const int i = threadIdx.x;
  if (i == 0) epoch_s = *epoch_counter + 1;
  __syncthreads();
  const int epoch = epoch_s;
  if (i < world) {
    int* dst = peer_signal[i] + rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
    const long long t0 = clock64();
    while (true) {
      int v;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(my_signal + i) : "memory");
      if (v >= epoch) break;
      if (clock64() - t0 > 20000000000LL) {  // ~10 s: report instead of hanging the GPU
        atomicExch(error_flag, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (i == 0) *epoch_counter = epoch;
}

// All-gather of n int32 per rank over peer memory, fused with a barrier: every
// rank writes its row into slot [rank] of every peer's (world, n) array, fences
// at system scope, then signals and waits like ipc_barrier_kernel. Graph safe
// (device epoch); doubles as "every rank has finished its previous step".
__global__ void ipc_allgather_kernel(const int32_t* __restrict__ src, int n,
                                     int32_t* const* __restrict__ peer_dst, int world, int rank,
                                     int* const* __restrict__ peer_signal, int* my_signal,
                                     int* epoch_counter, int* error_flag) {
  __shared__ int epoch_s;
  const int tid = threadIdx.x;
  for (int i = tid; i < n; i += blockDim.x) {
    const int32_t v = src[i];
    for (int p = 0; p < world; ++p) peer_dst[p][rank * n + i] = v;
  }
  __threadfence_system();
  if (tid == 0) epoch_s = *epoch_counter + 1;
  __syncthreads();
  const int epoch = epoch_s;
  if (tid < world) {
    int* dst = peer_signal[tid] + rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
    const long long t0 = clock64();
    while (true) {
      int v;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(my_signal + tid)
                   : "memory");
      if (v >= epoch) break;
      if (clock64() - t0 > 20000000000LL) {
        atomicExch(error_flag, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (tid == 0) *epoch_counter = epoch;
}

int launch_ipc_allgather(const int32_t* src, int n, int32_t* const* peer_dst, int world, int rank,
                         int* const* peer_signal, int* my_signal, int* epoch_counter,
                         int* error_flag, cudaStream_t st) {
  ipc_allgather_kernel<<<1, 256, 0, st>>>(src, n, peer_dst, world, rank, peer_signal, my_signal,
                                          epoch_counter, error_flag);
  return (int)cudaGetLastError();
}

// Source side of the return (k=1): out[t] = owner's combined row, loaded over
// NVLink from the owner's receive-layout buffer (16 B per lane, 512 B per warp
// access). Dropped tokens were already written (out = x) by the dispatch.
// dst[i] = src[index[i]]: the layout transforms between the phases of the
// hierarchical / coordinated exchanges (warp per row, 16-B vectors).
__global__ void gather_rows_kernel(const uint4* __restrict__ src, int64_t vec_per_row,
                                   const int32_t* __restrict__ index, int64_t n,
                                   uint4* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += warps_total) {
    const uint4* s = src + (int64_t)index[i] * vec_per_row;
    uint4* d = dst + i * vec_per_row;
    for (int64_t v = lane; v < vec_per_row; v += 32) d[v] = __ldg(s + v);
  }
}

int launch_gather_rows(const uint8_t* src, int64_t row_bytes, const int32_t* index, int64_t n,
                       uint8_t* dst, cudaStream_t st) {
  int64_t blocks = (n + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  gather_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(src),
                                                       row_bytes / 16, index, n,
                                                       reinterpret_cast<uint4*>(dst));
  return (int)cudaGetLastError();
}

template <typename V>
__global__ void pull_rows_kernel(int64_t S, int64_t row_bytes, int k, int e_per_rank,
                                 const int32_t* __restrict__ ids,
                                 const int32_t* __restrict__ row_index,
                                 uint8_t* const* __restrict__ peer_rows, uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t nvec = row_bytes / (int64_t)sizeof(V);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < S;
       t += warps_total) {
    const int32_t r = row_index[t * k];
    if (r < 0) continue;
    const V* src = reinterpret_cast<const V*>(peer_rows[ids[t * k] / e_per_rank] +
                                              (int64_t)r * row_bytes);
    V* dst = reinterpret_cast<V*>(out + t * row_bytes);
    constexpr int U = 4;
    int64_t i = lane;
    for (; i + 32 * (U - 1) < nvec; i += 32 * U) {
      V v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = src[i + 32 * u];
#pragma unroll
      for (int u = 0; u < U; ++u) dst[i + 32 * u] = v[u];
    }
    for (; i < nvec; i += 32) dst[i] = src[i];
  }
}

int launch_pull_rows(int64_t S, int64_t row_bytes, int k, int e_per_rank, const int32_t* ids,
                     const int32_t* row_index, uint8_t* const* peer_rows, uint8_t* out,
                     cudaStream_t st) {
  if (S == 0) return 0;
  int64_t g = (S + 7) / 8;
  if (g > 148 * 64) g = 148 * 64;
  if (comm_block_limit() > 0 && g > comm_block_limit()) g = comm_block_limit();
  if (row_bytes % 16 == 0)
    pull_rows_kernel<uint4><<<(unsigned)g, 256, 0, st>>>(S, row_bytes, k, e_per_rank, ids,
                                                         row_index, peer_rows, out);
  else
    pull_rows_kernel<uint16_t><<<(unsigned)g, 256, 0, st>>>(S, row_bytes, k, e_per_rank, ids,
                                                            row_index, peer_rows, out);
  return (int)cudaGetLastError();
}

int launch_ep_plan(const int32_t* counts, int world, int rank, int E, int C, int64_t cap,
                   int32_t* slot_base, int32_t* row_base, int32_t* seg_start, int32_t* seg_rows,
                   int32_t* recv_rows, cudaStream_t st, int padded) {
  const size_t smem = ((size_t)world * C * E + (size_t)world * C) * sizeof(int);
  if (smem > 48 * 1024 || (padded && C != 1)) return MOE_EINVAL;
  ep_plan_kernel<<<1, 256, smem, st>>>(counts, world, rank, E, C, cap, slot_base, row_base,
                                       seg_start, seg_rows, recv_rows, padded);
  return (int)cudaGetLastError();
}

int launch_ipc_barrier(int* const* peer_signal, int* my_signal, int world, int rank,
                       int* epoch_counter, int* error_flag, cudaStream_t st) {
  ipc_barrier_kernel<<<1, 32, 0, st>>>(peer_signal, my_signal, world, rank, epoch_counter,
                                       error_flag);
  return (int)cudaGetLastError();
}

}  // namespace moe

#define CHECK(cond)                 \
  do {                              \
    if (!(cond)) return MOE_EINVAL; \
  } while (0)

extern "C" {

int moe_ipc_malloc(size_t bytes, void** ptr) {
  CHECK(ptr && bytes > 0);
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaMemset(*ptr, 0, bytes);
}

int moe_ipc_free(void* ptr) { return ptr ? (int)cudaFree(ptr) : MOE_OK; }

int moe_enable_peer_access(int peer_device) {
  CHECK(peer_device >= 0);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return MOE_OK;
  }
  return (int)e;
}

int moe_ipc_get_handle(void* ptr, void* handle64) {
  CHECK(ptr && handle64);
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return (int)e;
  memcpy(handle64, &h, sizeof(h));
  return MOE_OK;
}

int moe_ipc_open_handle(const void* handle64, void** ptr) {
  CHECK(ptr && handle64);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  return (int)cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
}

int moe_ipc_close_handle(void* ptr) { return ptr ? (int)cudaIpcCloseMemHandle(ptr) : MOE_OK; }

int moe_ep_plan(const int32_t* counts, int world, int rank, int E, int64_t cap, int32_t* slot_base,
                int32_t* row_base, int32_t* seg_start, int32_t* seg_rows, int32_t* recv_rows,
                void* stream) {
  CHECK(world >= 1 && rank >= 0 && rank < world && E >= world && E % world == 0 && cap >= 0);
  CHECK(counts && slot_base && row_base && seg_start && seg_rows && recv_rows);
  return moe::launch_ep_plan(counts, world, rank, E, 1, cap, slot_base, row_base, seg_start,
                             seg_rows, recv_rows, reinterpret_cast<cudaStream_t>(stream));
}

int moe_ep_plan_padded(const int32_t* counts, int world, int rank, int E, int64_t cap,
                       int32_t* slot_base, int32_t* row_base, int32_t* seg_start, int32_t* seg_rows,
                       int32_t* recv_rows, void* stream) {
  CHECK(world >= 1 && rank >= 0 && rank < world && E >= world && E % world == 0 && cap >= 0);
  CHECK((int64_t)(E / world) * cap < ((int64_t)1 << 31));
  CHECK(counts && slot_base && row_base && seg_start && seg_rows && recv_rows);
  return moe::launch_ep_plan(counts, world, rank, E, 1, cap, slot_base, row_base, seg_start,
                             seg_rows, recv_rows, reinterpret_cast<cudaStream_t>(stream), 1);
}

int moe_ep_plan_chunked(const int32_t* counts, int world, int rank, int E, int chunks, int64_t cap,
                        int32_t* slot_base, int32_t* row_base, int32_t* seg_start,
                        int32_t* seg_rows, int32_t* recv_rows, void* stream) {
  CHECK(world >= 1 && rank >= 0 && rank < world && E >= world && E % world == 0 && cap >= 0 &&
        chunks >= 1 && chunks <= 64);
  CHECK(counts && slot_base && row_base && seg_start && seg_rows && recv_rows);
  return moe::launch_ep_plan(counts, world, rank, E, chunks, cap, slot_base, row_base, seg_start,
                             seg_rows, recv_rows, reinterpret_cast<cudaStream_t>(stream));
}

int moe_set_launch_limits(int gemm_ctas, int comm_blocks) {
  CHECK(gemm_ctas >= 0 && comm_blocks >= 0);
  moe::set_launch_limits(gemm_ctas, comm_blocks);
  return MOE_OK;
}

int moe_ipc_barrier(int* const* peer_signal, int* my_signal, int world, int rank,
                    int* epoch_counter, int* error_flag, void* stream) {
  CHECK(world >= 1 && world <= 32 && rank >= 0 && rank < world);
  CHECK(peer_signal && my_signal && epoch_counter && error_flag);
  return moe::launch_ipc_barrier(peer_signal, my_signal, world, rank, epoch_counter, error_flag,
                                 reinterpret_cast<cudaStream_t>(stream));
}

int moe_ipc_allgather_i32(const int32_t* src, int n, int32_t* const* peer_dst, int world, int rank,
                          int* const* peer_signal, int* my_signal, int* epoch_counter,
                          int* error_flag, void* stream) {
  CHECK(n >= 1 && world >= 1 && world <= 32 && rank >= 0 && rank < world);
  CHECK(src && peer_dst && peer_signal && my_signal && epoch_counter && error_flag);
  return moe::launch_ipc_allgather(src, n, peer_dst, world, rank, peer_signal, my_signal,
                                   epoch_counter, error_flag, reinterpret_cast<cudaStream_t>(stream));
}

int moe_dispatch_p2p(const void* x, int64_t S, int64_t row_bytes, int E, int k, int64_t cap,
                     const int32_t* ids, const int32_t* local_rank, const int32_t* tile_offsets,
                     const float* gate_probs, const int32_t* slot_base, const int32_t* row_base,
                     int e_per_rank, void* const* peer_recv, int32_t* const* peer_token,
                     float* const* peer_prob, int32_t* slots, int32_t* row_index,
                     void* out_dropped, int32_t* const* peer_src, int my_rank, void* stream) {
  CHECK(S >= 0 && row_bytes >= 0 && row_bytes % 2 == 0 && E >= 1 && (k == 1 || k == 2) &&
        cap >= 0 && e_per_rank >= 1);
  if (S == 0) return MOE_OK;
  CHECK(x && ids && local_rank && tile_offsets && gate_probs && slot_base && row_base &&
        peer_recv && peer_token && peer_prob && slots && row_index);
  moe::ScatterArgs a;
  a.x = static_cast<const uint8_t*>(x);
  a.S = S, a.row_bytes = row_bytes, a.k = k, a.E = E, a.cap = cap;
  a.ids = ids, a.slots = slots, a.local_rank = local_rank, a.tile_offsets = tile_offsets;
  a.gate_probs = gate_probs;
  a.slot_base = slot_base, a.row_base = row_base;
  a.peer_buf = reinterpret_cast<uint8_t* const*>(peer_recv);
  a.peer_token = peer_token, a.peer_prob = peer_prob, a.e_per_rank = e_per_rank;
  a.out_dropped = static_cast<uint8_t*>(out_dropped);
  a.row_index = row_index;
  a.peer_src = peer_src;
  a.my_rank = my_rank;
  return moe::launch_scatter(a, reinterpret_cast<cudaStream_t>(stream));
}

int moe_gather_rows(const void* src, int64_t row_bytes, const int32_t* index, int64_t n,
                    void* dst, void* stream) {
  CHECK(row_bytes >= 16 && row_bytes % 16 == 0 && n >= 0);
  if (n == 0) return MOE_OK;
  CHECK(src && index && dst && src != dst);
  return moe::launch_gather_rows(static_cast<const uint8_t*>(src), row_bytes, index, n,
                                 static_cast<uint8_t*>(dst), reinterpret_cast<cudaStream_t>(stream));
}

int moe_pull_rows_p2p(int64_t S, int64_t row_bytes, int E, int k, const int32_t* ids,
                      const int32_t* row_index, int e_per_rank, void* const* peer_rows, void* out,
                      void* stream) {
  CHECK(S >= 0 && row_bytes >= 0 && row_bytes % 2 == 0 && E >= 1 && k == 1 && e_per_rank >= 1);
  if (S == 0) return MOE_OK;
  CHECK(ids && row_index && peer_rows && out);
  return moe::launch_pull_rows(S, row_bytes, k, e_per_rank, ids, row_index,
                               reinterpret_cast<uint8_t* const*>(peer_rows),
                               static_cast<uint8_t*>(out), reinterpret_cast<cudaStream_t>(stream));
}

int moe_grouped_gemm_bf16_combine_rows(const void* A, int64_t a_rows, int K, const void* B,
                                       int64_t b_rows, int N, const float* bias, int num_groups,
                                       const int32_t* row_start, const int32_t* rows,
                                       const int32_t* weight_idx, int64_t max_group_rows,
                                      const int32_t* row_token, const float* row_prob,
                                      const void* x_rows, void* out_rows, void* stream) {
  CHECK(a_rows >= 0 && K >= 8 && K % 8 == 0 && N >= 1 && b_rows >= N && num_groups >= 1);
  CHECK(max_group_rows >= 0);
  if (a_rows == 0 || max_group_rows == 0) return MOE_OK;
  CHECK(A && B && row_start && rows && row_token && row_prob && x_rows && out_rows);
  return moe::launch_grouped_gemm_bf16(A, a_rows, K, B, b_rows, N, bias, nullptr, num_groups,
                                       row_start, 0, rows, 0, weight_idx, max_group_rows, 2,
                                       reinterpret_cast<cudaStream_t>(stream), row_token, row_prob,
                                       x_rows, out_rows, 1);
}

int moe_grouped_gemm_bf16_push(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                               int N, const float* bias, int num_groups, const int32_t* row_start,
                               int64_t row_stride, const int32_t* rows, const int32_t* weight_idx,
                               int64_t max_group_rows, int combine, const int32_t* row_token,
                               const float* row_prob, const int32_t* row_src,
                               void* const* push_base, const void* x_rows, void* stream) {
  CHECK(a_rows >= 0 && K >= 8 && K % 8 == 0 && N >= 1 && b_rows >= N && num_groups >= 1);
  CHECK(max_group_rows >= 0 && (combine == 0 || combine == 1));
  if (a_rows == 0 || max_group_rows == 0) return MOE_OK;
  CHECK(A && B && (row_start || row_stride > 0) && rows && row_token && row_src && push_base);
  if (combine) CHECK(row_prob && x_rows);
  // combine = 1: act 2 (EPI_BIAS_COMBINE, x = the receive row itself); 0: bias only
  return moe::launch_grouped_gemm_bf16(A, a_rows, K, B, b_rows, N, bias, nullptr, num_groups,
                                       row_start, row_start ? 0 : row_stride, rows, 0, weight_idx,
                                       max_group_rows, combine ? 2 : 0,
                                       reinterpret_cast<cudaStream_t>(stream),
                                       row_token, row_prob, x_rows, nullptr, combine ? 1 : 0, 0,
                                       nullptr, push_base, row_src);
}

}  // extern "C"
