// Streaming-read probe: how fast can one CTA per SM pull a row-major bf16
// matrix (65536 x 2048, 268 MB, the C3 gate's x) into shared memory, 128-row
// units x 64-column k-blocks (the gate's A-tile order), with no compute?
//   mode 0  TMA 2-D box 64 x 128 (SWIZZLE_128B), one producer thread, STAGES ring
//   mode 1  cp.async 16 B by 4 loader warps into the same swizzled layout,
//           completion through cp.async.mbarrier.arrive.noinc
//   mode 2  plain LDG 16 B by 4 warps into registers (no smem), the same order
//   mode 3  TMA 1-D bulk copies of 16 KB contiguous (4 whole rows per k-block)
//   mode 4  mode 0 with the consumer holding every stage `hold` SM cycles before
//           freeing it (stands in for the MMA -> commit latency of the gate)
// One consumer warp per CTA waits each stage and frees it (modes 0, 1, 3).
// L2 is flushed (512 MB write) before every launch; median of 20 launches.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        -I paper_2201_05596_b200/csrc tools/stream_probe.cu -o tools/stream_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace moe;

constexpr int kRows = 65536, kCols = 2048, kUnit = 128, kBK = 64;
constexpr int kStageBytes = kUnit * kBK * 2;  // 16 KB
constexpr int kKB = kCols / kBK;              // 32 k-blocks per unit
constexpr int kUnits = kRows / kUnit;         // 512

template <int MODE, int STAGES>
__global__ void __launch_bounds__(192, 1)
    stream_kernel(const __grid_constant__ CUtensorMap map, const __nv_bfloat16* x,
                  unsigned long long* sink, long long* cycles, int hold) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], MODE == 1 ? 128 : 1);
      mbar_init(&empty[s], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  unsigned long long acc = 0;
  if (MODE == 2) {
    if (warp >= 1 && warp <= 4) {
      const int w = warp - 1;
      for (int u = blockIdx.x; u < kUnits; u += gridDim.x) {
        for (int kb = 0; kb < kKB; ++kb) {
          uint4 v[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {  // warp: rows w*32 + 4i .. +3, 128 B each
            const int r = u * kUnit + w * 32 + 4 * i + lane / 8;
            v[i] = __ldg(reinterpret_cast<const uint4*>(x + (size_t)r * kCols + kb * kBK) + (lane % 8));
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) acc += (unsigned long long)v[i].x + v[i].y + v[i].z + v[i].w;
        }
      }
    }
  } else if (warp == 0) {
    // producer(s)
    if (MODE == 0 || MODE == 3 || MODE == 4) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < kUnits; u += gridDim.x) {
        for (int kb = 0; kb < kKB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[stage], kStageBytes);
            if (MODE == 0 || MODE == 4)
              tma_load_2d(smem + stage * kStageBytes, &map, &full[stage], kb * kBK, u * kUnit);
            else
              bulk_load(smem + stage * kStageBytes,
                        x + (size_t)u * kUnit * kCols + (size_t)kb * (kStageBytes / 2), kStageBytes,
                        &full[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // consumer
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < kUnits; u += gridDim.x) {
      for (int kb = 0; kb < kKB; ++kb) {
        mbar_wait(&full[stage], phase);
        if (lane == 0) {
          acc ^= *reinterpret_cast<volatile unsigned long long*>(smem + stage * kStageBytes + 8 * (kb & 7));
          if (MODE == 4) {  // hold the stage (in flight, like an MMA reading it)
            const long long t = clock64();
            while (clock64() - t < hold) {
            }
          }
          mbar_arrive(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (MODE == 1 && warp >= 2 && warp <= 5) {
    const int w = warp - 2;
    int stage = 0;
    uint32_t phase = 0;
    for (int u = blockIdx.x; u < kUnits; u += gridDim.x) {
      for (int kb = 0; kb < kKB; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* dst = smem + stage * kStageBytes;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = w * 32 + 4 * i + lane / 8, c = lane % 8;
          const __nv_bfloat16* src = x + (size_t)(u * kUnit + rr) * kCols + kb * kBK + c * 8;
          const uint32_t d = smem_u32(dst + rr * 128 + ((c ^ (rr & 7)) * 16));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[stage]))
                     : "memory");
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  }
  if (acc == 0x123456789ull) sink[0] = acc;
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int MODE, int STAGES>
static void run(const CUtensorMap& map, const __nv_bfloat16* x, uint8_t* flush, unsigned long long* sink,
                long long* cyc, int grid, int hold = 0) {
  const int smem = STAGES * kStageBytes + 1024;
  cudaFuncSetAttribute(stream_kernel<MODE, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ts;
  std::vector<long long> hc(grid);
  long long cmax = 0;
  for (int it = 0; it < 23; ++it) {
    cudaMemsetAsync(flush, it & 0xff, 512ull << 20);
    cudaEventRecord(e0);
    stream_kernel<MODE, STAGES><<<grid, 192, smem>>>(map, x, sink, cyc, hold);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 3) ts.push_back(ms * 1e3f);
    cudaMemcpy(hc.data(), cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    if (it >= 3) cmax = std::max(cmax, *std::max_element(hc.begin(), hc.end()));
  }
  cudaError_t err = cudaGetLastError();
  std::sort(ts.begin(), ts.end());
  const float us = ts[ts.size() / 2];
  const double bytes = (double)kRows * kCols * 2;
  const double per_sm = bytes / grid;
  printf("mode %d hold %5d stages %2d grid %3d  %7.1f us  %6.0f GB/s  max CTA %6.1f kcycles  %5.1f B/clk/SM%s\n",
         MODE, hold, STAGES, grid, us, bytes / us / 1e3, cmax / 1e3,
         per_sm * ((double)((kUnits + grid - 1) / grid) / ((double)kUnits / grid)) / cmax,
         err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
  __nv_bfloat16* x;
  uint8_t* flush;
  unsigned long long* sink;
  long long* cyc;
  cudaMalloc(&x, (size_t)kRows * kCols * 2);
  cudaMemset(x, 1, (size_t)kRows * kCols * 2);
  cudaMalloc(&flush, 512ull << 20);
  cudaMalloc(&sink, 8);
  cudaMalloc(&cyc, 1024 * sizeof(long long));
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)kCols, (cuuint64_t)kRows};
  cuuint64_t strides[1] = {(cuuint64_t)kCols * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kUnit};
  cuuint32_t es[2] = {1, 1};
  CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    return 1;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int grid : {sms}) {
    run<0, 8>(map, x, flush, sink, cyc, grid);
    run<1, 8>(map, x, flush, sink, cyc, grid);
    run<2, 8>(map, x, flush, sink, cyc, grid);
    run<3, 8>(map, x, flush, sink, cyc, grid);
    // ring depth: an MMA that holds each stage until it completes shortens the
    // effective ring (mode 0 with fewer stages)
    run<0, 2>(map, x, flush, sink, cyc, grid);
    run<0, 3>(map, x, flush, sink, cyc, grid);
    run<0, 4>(map, x, flush, sink, cyc, grid);
    run<0, 6>(map, x, flush, sink, cyc, grid);
    for (int hold : {100, 200, 400}) run<4, 8>(map, x, flush, sink, cyc, grid, hold);
  }
  return 0;
}
