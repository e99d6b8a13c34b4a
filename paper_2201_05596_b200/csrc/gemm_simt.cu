// fp32 SIMT grouped GEMM: the parity path for fp32 layers (BASELINE config 1).
// tcgen05 has no true-fp32 kind (kind::tf32 would miss rtol 1e-5), so fp32
// runs on CUDA cores with fp32 accumulation and an accurate tanhf GELU.
//
//   D[rows of g] = act(A[rows of g] (r x K) . B_w(g) (K x N) + bias_w(g))
//
// B keeps the reference layout w1 (M, 4M) / w2 (4M, M) (arch.py:347-354).
#include "common.cuh"
#include "moe_kernels.h"

namespace moe {

constexpr int SBM = 128, SBN = 128, SBK = 16;

template <int ACT>
__global__ void __launch_bounds__(256) gemm_f32_simt_kernel(
    const float* __restrict__ A, int K, const float* __restrict__ B, int N,
    const float* __restrict__ bias, float* __restrict__ D, const int32_t* __restrict__ row_start,
    int64_t row_stride, const int32_t* __restrict__ rows, int64_t rows_const,
    const int32_t* __restrict__ weight_idx) {
  __shared__ float As[SBK][SBM + 4];
  __shared__ float Bs[SBK][SBN + 4];
  const int g = blockIdx.z;
  const int64_t rows_g = rows ? rows[g] : rows_const;
  const int64_t m0 = (int64_t)blockIdx.y * SBM;
  if (m0 >= rows_g) return;
  const int n0 = blockIdx.x * SBN;
  const int64_t rs = row_start ? row_start[g] : (int64_t)g * row_stride;
  const int w = weight_idx ? weight_idx[g] : g;
  const float* Bw = B + (int64_t)w * K * N;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += SBK) {
#pragma unroll
    for (int p = 0; p < (SBM * SBK) / 256; ++p) {
      const int i = tid + 256 * p;
      const int r = i / SBK, kk = i % SBK;
      const int64_t row = m0 + r;
      float v = 0.f;
      if (row < rows_g && k0 + kk < K) v = A[(rs + row) * K + k0 + kk];
      As[kk][r] = v;
    }
#pragma unroll
    for (int p = 0; p < (SBK * SBN) / 256; ++p) {
      const int i = tid + 256 * p;
      const int kk = i / SBN, n = i % SBN;
      float v = 0.f;
      if (k0 + kk < K && n0 + n < N) v = Bw[(int64_t)(k0 + kk) * N + n0 + n];
      Bs[kk][n] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SBK; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = m0 + ty + 16 * i;
    if (row >= rows_g) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (bias) v += bias[(int64_t)w * N + n];
      if (ACT == 1) v = gelu_tanh_accurate(v);
      D[(rs + row) * N + n] = v;
    }
  }
}

int launch_grouped_gemm_f32(const float* A, int K, const float* B, int N, const float* bias,
                            float* D, int G, const int32_t* row_start, int64_t row_stride,
                            const int32_t* rows, int64_t rows_const, const int32_t* weight_idx,
                            int64_t max_group_rows, int act, cudaStream_t st) {
  if (G < 1 || K < 1 || N < 1) return MOE_EINVAL;
  if (max_group_rows == 0) return 0;
  dim3 grid((N + SBN - 1) / SBN, (unsigned)((max_group_rows + SBM - 1) / SBM), G);
  if (act == 1)
    gemm_f32_simt_kernel<1><<<grid, 256, 0, st>>>(A, K, B, N, bias, D, row_start, row_stride, rows,
                                                  rows_const, weight_idx);
  else
    gemm_f32_simt_kernel<0><<<grid, 256, 0, st>>>(A, K, B, N, bias, D, row_start, row_stride, rows,
                                                  rows_const, weight_idx);
  return (int)cudaGetLastError();
}

}  // namespace moe
