// Backward of the MoE layer forward, bf16 device path.
//
// The reference forward is tape-aware (arch.py:375-377): gradients flow through
// the gate probabilities that scale each expert's contribution (row_softmax,
// tensor.py:254-268, and take_elems, :271-292), not through the routing
// decisions. With out = x + sum_kept p_te * y_e(x_t) [+ shared(x)]:
//   dY_e[row]   = p * dOut[t]                         (mul vjp, tensor.py:191-207)
//   dp[t, j]    = <dOut[t], y_e[row]>                  (take_elems vjp)
//   dlogits[t]  = s_t * (g_t - <g_t, s_t>)            (row_softmax vjp, tensor.py:263-266)
//   dx[t]       = dOut[t] + sum_j dX_e[row] + dlogits[t] @ W_g^T [+ shared]
// The GEMMs run on the tcgen05 grouped kernel. Weight gradients contract over
// the token dimension: the kernel's weight-gradient mode reads both operands
// MN-major straight from the saved row-major activations (no transposes), with
// K = each expert's kept rows; bias gradients are column sums (colsum_rows_kernel).
#include "common.cuh"
#include "moe_kernels.h"

namespace moe {

// warp per token: dY rows (bf16) for kept assignments and dp (fp32)
__global__ void combine_bwd_kernel(const __nv_bfloat16* __restrict__ dout,
                                   const __nv_bfloat16* __restrict__ y, int64_t S, int M, int k,
                                   int64_t cap, const int32_t* __restrict__ ids,
                                   const int32_t* __restrict__ slots,
                                   const float* __restrict__ gp, __nv_bfloat16* __restrict__ dy,
                                   float* __restrict__ dp) {
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < S;
       t += warps_total) {
    const __nv_bfloat16* g = dout + t * M;
    for (int j = 0; j < k; ++j) {
      const int s = slots[t * k + j];
      if (s < 0) {
        if (lane == 0) dp[t * k + j] = 0.f;
        continue;
      }
      const int64_t row = (int64_t)ids[t * k + j] * cap + s;
      const float p = gp[t * k + j];
      const __nv_bfloat16* yr = y + row * M;
      __nv_bfloat16* dr = dy + row * M;
      float acc = 0.f;
      for (int c = lane * 2; c < M; c += 64) {  // M even
        const __nv_bfloat162 g2 = *reinterpret_cast<const __nv_bfloat162*>(g + c);
        const __nv_bfloat162 y2 = *reinterpret_cast<const __nv_bfloat162*>(yr + c);
        const float g0 = __low2float(g2), g1 = __high2float(g2);
        acc = fmaf(g0, __low2float(y2), acc);
        acc = fmaf(g1, __high2float(y2), acc);
        *reinterpret_cast<__nv_bfloat162*>(dr + c) = __floats2bfloat162_rn(p * g0, p * g1);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) dp[t * k + j] = acc;
    }
  }
}

// warp per token: dlogits = s * (g - <g, s>), g sparse at the kept choices.
// Output bf16 (S, Epad), zero in the padding columns; with split, rows are
// (2*Epad) = [hi | lo], hi + lo carrying ~16 mantissa bits: the gate term of dx
// is a large quantity that cancels against the expert term, so one bf16
// rounding of dlogits is visible in dx (K = 2*Epad GEMM against [Wg | Wg]).
__global__ void gate_bwd_kernel(const float* __restrict__ logits, int64_t S, int E, int Epad,
                                int k, const int32_t* __restrict__ ids,
                                const int32_t* __restrict__ slots, const float* __restrict__ dp,
                                __nv_bfloat16* __restrict__ dlogits, int split) {
  const int64_t ld = split ? 2 * (int64_t)Epad : Epad;
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < S;
       t += warps_total) {
    const float* lr = logits + t * E;
    float m = -INFINITY;
    for (int e = lane; e < E; e += 32) m = fmaxf(m, lr[e]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float sum = 0.f;
    for (int e = lane; e < E; e += 32) sum += expf(lr[e] - m);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    const float inv = 1.f / sum;
    // <g, s> over the k kept choices
    int ej[2] = {-1, -1};
    float gj[2] = {0.f, 0.f};
    float dot = 0.f;
    for (int j = 0; j < k; ++j) {
      if (slots[t * k + j] >= 0) {
        ej[j] = ids[t * k + j];
        gj[j] = dp[t * k + j];
        dot += gj[j] * expf(lr[ej[j]] - m) * inv;
      }
    }
    for (int e = lane; e < Epad; e += 32) {
      float v = 0.f;
      if (e < E) {
        const float se = expf(lr[e] - m) * inv;
        const float ge = (e == ej[0] ? gj[0] : 0.f) + (e == ej[1] ? gj[1] : 0.f);
        v = se * (ge - dot);
      }
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      dlogits[t * ld + e] = hi;
      if (split) dlogits[t * ld + Epad + e] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
  }
}

// out[g][c] += sum over rows r < rows_g of X[g*row_stride + r][c] (fp32): bias
// gradients. Block = 32 x 8 threads over 256 columns (8 per thread, 16-B loads);
// blockIdx.z splits the rows, one atomic per column per block.
__global__ void colsum_rows_kernel(const __nv_bfloat16* __restrict__ X, int W, int64_t row_stride,
                                   const int32_t* __restrict__ rows, int64_t rows_const,
                                   float* __restrict__ out) {
  __shared__ float part[8][256 + 4];
  const int g = blockIdx.y;
  const int64_t rg = rows ? rows[g] : rows_const;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int c = blockIdx.x * 256 + tx * 8;
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  if (c < W) {
    const __nv_bfloat16* Xg = X + (int64_t)g * row_stride * W + c;
    for (int64_t r = (int64_t)blockIdx.z * 8 + ty; r < rg; r += (int64_t)gridDim.z * 8) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(Xg + r * W));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        acc[2 * i] += f.x;
        acc[2 * i + 1] += f.y;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) part[ty][tx * 8 + i] = acc[i];
  __syncthreads();
  const int j = ty * 32 + tx;  // 256 columns, one per thread
  float v = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) v += part[i][j];
  const int col = blockIdx.x * 256 + j;
  if (col < W && v != 0.f) atomicAdd(&out[(int64_t)g * W + col], v);
}

// dx[t] = dout[t] + sum_j kept dXr[row_j] + extra1[t] (+ extra2[t])
__global__ void bwd_dx_kernel(const __nv_bfloat16* __restrict__ dout,
                              const __nv_bfloat16* __restrict__ dxr, int64_t S, int M, int k,
                              int64_t cap, const int32_t* __restrict__ ids,
                              const int32_t* __restrict__ slots,
                              const __nv_bfloat16* __restrict__ extra1,
                              const __nv_bfloat16* __restrict__ extra2,
                              __nv_bfloat16* __restrict__ dx) {
  // half-warp per token, 16-B vectors (M % 8 == 0); fp32 sum in the order
  // dout + dX_e0 + dX_e1 + extra1 + extra2
  constexpr int LPT = 16;
  const int lane = threadIdx.x & (LPT - 1);
  const int64_t slots_total = (int64_t)gridDim.x * (blockDim.x >> 5) * 2;
  for (int64_t t = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 2 +
                   (threadIdx.x & 31) / LPT;
       t < S; t += slots_total) {
    int64_t rr[2] = {-1, -1};
    for (int j = 0; j < k; ++j) {
      const int s = slots[t * k + j];
      if (s >= 0) rr[j] = (int64_t)ids[t * k + j] * cap + s;
    }
    for (int c = lane * 8; c < M; c += LPT * 8) {
      float v[8];
      auto acc = [&](const __nv_bfloat16* p, bool first) {
        const uint4 q = *reinterpret_cast<const uint4*>(p);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          v[2 * i] = first ? f.x : v[2 * i] + f.x;
          v[2 * i + 1] = first ? f.y : v[2 * i + 1] + f.y;
        }
      };
      acc(dout + t * M + c, true);
      for (int j = 0; j < 2; ++j)
        if (rr[j] >= 0) acc(dxr + rr[j] * M + c, false);
      if (extra1) acc(extra1 + t * M + c, false);
      if (extra2) acc(extra2 + t * M + c, false);
      uint4 o;
      uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        op[i] = *reinterpret_cast<const uint32_t*>(&b);
      }
      *reinterpret_cast<uint4*>(dx + t * M + c) = o;
    }
  }
}

static int grid_warps(int64_t S) {
  int64_t g = (S + 7) / 8;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace moe

#define CHECK(cond)                 \
  do {                              \
    if (!(cond)) return MOE_EINVAL; \
  } while (0)

extern "C" {

int moe_combine_bwd_bf16(const void* dout, const void* y, int64_t S, int M, int E, int k,
                         int64_t cap, const int32_t* ids, const int32_t* slots,
                         const float* gate_probs, void* dy, float* dp, void* stream) {
  CHECK(S >= 0 && M >= 2 && M % 2 == 0 && E >= 1 && (k == 1 || k == 2) && cap >= 0);
  if (S == 0) return MOE_OK;
  CHECK(dout && ids && slots && gate_probs && dp && (cap == 0 || (y && dy)));
  moe::combine_bwd_kernel<<<moe::grid_warps(S), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (const __nv_bfloat16*)dout, (const __nv_bfloat16*)y, S, M, k, cap, ids, slots, gate_probs,
      (__nv_bfloat16*)dy, dp);
  return (int)cudaGetLastError();
}

int moe_gate_bwd(const float* logits, int64_t S, int E, int Epad, int k, const int32_t* ids,
                 const int32_t* slots, const float* dp, void* dlogits, int split, void* stream) {
  CHECK(S >= 0 && E >= 1 && Epad >= E && (k == 1 || k == 2) && (split == 0 || split == 1));
  if (S == 0) return MOE_OK;
  CHECK(logits && ids && slots && dp && dlogits);
  moe::gate_bwd_kernel<<<moe::grid_warps(S), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      logits, S, E, Epad, k, ids, slots, dp, (__nv_bfloat16*)dlogits, split);
  return (int)cudaGetLastError();
}

int moe_colsum_rows_bf16(const void* X, int W, int num_groups, int64_t row_stride,
                         const int32_t* rows, int64_t rows_const, float* out, void* stream) {
  CHECK(W >= 8 && W % 8 == 0 && num_groups >= 1 && num_groups <= 65535 && row_stride >= 0 &&
        rows_const >= 0);
  CHECK(X && out);
  const int64_t max_rows = rows ? (row_stride > 0 ? row_stride : rows_const) : rows_const;
  if (max_rows == 0) return MOE_OK;
  const int nx = (W + 255) / 256;
  int64_t splits = (4 * 148 + (int64_t)nx * num_groups - 1) / ((int64_t)nx * num_groups);
  splits = splits < 1 ? 1 : splits;
  const int64_t by_rows = (max_rows + 63) / 64;
  if (splits > by_rows) splits = by_rows;
  if (splits > 65535) splits = 65535;
  dim3 grid(nx, num_groups, (unsigned)splits);
  moe::colsum_rows_kernel<<<grid, dim3(32, 8), 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (const __nv_bfloat16*)X, W, row_stride, rows, rows_const, out);
  return (int)cudaGetLastError();
}

int moe_grouped_gemm_bf16_wgrad(const void* X, int64_t x_rows, int P, const void* Y, int Q,
                                int num_groups, int64_t k_stride, const int32_t* k_rows,
                                int64_t k_rows_const, void* D, void* stream) {
  CHECK(x_rows >= 0 && P >= 8 && P % 8 == 0 && Q >= 8 && Q % 8 == 0 && num_groups >= 1 &&
        k_stride >= 0 && k_rows_const >= 0);
  CHECK(D && (x_rows == 0 || (X && Y)));
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (x_rows == 0)
    return (int)cudaMemsetAsync(D, 0, (size_t)num_groups * P * Q * 2, st);
  return moe::launch_wgrad_bf16(X, x_rows, P, Y, Q, num_groups, k_stride, k_rows, k_rows_const, D,
                                0, st);
}

int moe_gemm_bf16_wgrad_f32(const void* X, int64_t rows, int P, const void* Y, int Q, float* D,
                            void* stream) {
  CHECK(rows >= 0 && P >= 8 && P % 8 == 0 && Q >= 8 && Q % 8 == 0);
  CHECK(D && (rows == 0 || (X && Y)));
  if (rows == 0) return MOE_OK;
  // split K (the token rows) so the (P x Q) output tiles times the splits fill the SMs
  const int tm = Q <= 128 ? 128 : 256, bn = Q <= 128 ? 128 : 256;
  const int64_t tiles = (int64_t)((P + tm - 1) / tm) * ((Q + bn - 1) / bn);
  const int64_t ctas_per_tile = tm / 128;
  int64_t splits = (148 / ctas_per_tile + tiles - 1) / tiles;
  const int64_t max_splits = (rows + 255) / 256;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  const int64_t chunk = ((rows + splits - 1) / splits + 63) / 64 * 64;
  const int G = (int)((rows + chunk - 1) / chunk);
  // the last chunk reads past `rows`: TMA zero-fills out-of-bounds rows
  return moe::launch_wgrad_bf16(X, rows, P, Y, Q, G, chunk, nullptr, chunk, D, 1,
                                reinterpret_cast<cudaStream_t>(stream));
}

int moe_bwd_dx_bf16(const void* dout, const void* dxr, int64_t S, int M, int E, int k, int64_t cap,
                    const int32_t* ids, const int32_t* slots, const void* extra1,
                    const void* extra2, void* dx, void* stream) {
  CHECK(S >= 0 && M >= 8 && M % 8 == 0 && E >= 1 && (k == 1 || k == 2) && cap >= 0);
  if (S == 0) return MOE_OK;
  CHECK(dout && ids && slots && dx && (cap == 0 || dxr));
  moe::bwd_dx_kernel<<<(moe::grid_warps(S) + 1) / 2, 256, 0,
                       reinterpret_cast<cudaStream_t>(stream)>>>(
      (const __nv_bfloat16*)dout, (const __nv_bfloat16*)dxr, S, M, k, cap, ids, slots,
      (const __nv_bfloat16*)extra1, (const __nv_bfloat16*)extra2, (__nv_bfloat16*)dx);
  return (int)cudaGetLastError();
}

int moe_grouped_gemm_bf16_aux(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                              int N, const float* bias, void* D, int num_groups,
                              const int32_t* row_start, int64_t row_stride, const int32_t* rows,
                              int64_t rows_const, const int32_t* weight_idx,
                              int64_t max_group_rows, int act, void* aux, void* stream) {
  CHECK(a_rows >= 0 && K >= 8 && K % 8 == 0 && N >= 1 && b_rows >= N && num_groups >= 1);
  CHECK(act == MOE_ACT_GELU_SAVE || act == MOE_ACT_GELU_BWD);
  CHECK(max_group_rows >= 0 && rows_const >= 0);
  if (a_rows == 0 || max_group_rows == 0) return MOE_OK;
  CHECK(A && B && D && aux);
  const int internal = act == MOE_ACT_GELU_SAVE ? 3 : 4;
  return moe::launch_grouped_gemm_bf16(
      A, a_rows, K, B, b_rows, N, bias, D, num_groups, row_start, row_stride, rows, rows_const,
      weight_idx, max_group_rows, internal, reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr,
      act == MOE_ACT_GELU_BWD ? aux : nullptr, act == MOE_ACT_GELU_SAVE ? aux : nullptr, 0);
}

}  // extern "C"
