// Routing kernels for the MoE layer forward on sm_100a:
//   * top-k gate from logits (softmax + arg-max with lower-index ties)
//   * plan tiles  : per-128-token-tile local ranks + per-expert tile counts
//   * plan scan   : per-expert exclusive scan over tiles (+ EP rank offsets)
//   * plan slots  : slot = tile offset + local rank, DROPPED past capacity
//   * int64 exclusive scan and the Blelloch tree-order f64 scan
//   * table-driven scatter (dispatch) and combine
//
// Reference semantics: /root/reference/pkg/src/moekit/gating.py:142-307 and
// arch.py:372-413. All integer outputs are bit-exact with the reference.
#include "common.cuh"
#include "moe_kernels.h"

#include <atomic>
#include <cstdlib>

namespace moe {

// MOE_PDL=1: programmatic dependent launch for the forward hot-path kernels.
// Parity-green (full GPU suite) but no gain: C2 / C4 within noise, C3 burst
// 17.1 vs 17.5 M tok/s (profiles/r2_ab_pdl.log) - off by default
bool pdl_on() {
  static const bool on = [] {
    const char* v = getenv("MOE_PDL");
    return v ? atoi(v) != 0 : false;
  }();
  return on;
}

// ============================================================ top-k gate
// One warp per token row. Lane l owns columns l, l+32, ... (coalesced).
constexpr int kNoExpert = 0x7fffffff;

// Order of np.argsort(-logits, kind="stable") (gating.py:159-161): descending
// value, ties to the lower expert index, NaN after every number (numpy sorts
// NaN last) - so a row of NaN / -inf still routes to valid expert indices.
template <typename T>
MOE_DEV bool ranks_before(T v, int i, T bv, int bi) {
  if (i == kNoExpert) return false;
  if (bi == kNoExpert) return true;
  const bool vn = v != v, bn = bv != bv;
  if (vn != bn) return bn;
  if (!vn && v != bv) return v > bv;
  return i < bi;
}

template <typename T>
MOE_DEV void better(T v, int i, T& bv, int& bi) {
  if (ranks_before(v, i, bv, bi)) {
    bv = v;
    bi = i;
  }
}

template <typename T>
MOE_DEV void warp_argmax(T& v, int& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    T ov = __shfl_xor_sync(0xffffffffu, v, off);
    int oi = __shfl_xor_sync(0xffffffffu, i, off);
    better(ov, oi, v, i);
  }
}

MOE_DEV float exp_t(float x) { return expf(x); }
MOE_DEV double exp_t(double x) { return exp(x); }

template <typename T>
__global__ void topk_gate_kernel(const T* __restrict__ logits, int64_t S, int E, int k,
                                 int32_t* __restrict__ ids, T* __restrict__ gate_probs,
                                 T* __restrict__ probs) {
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < S;
       t += warps_total) {
    const T* row = logits + t * E;
    const T ninf = -INFINITY;
    T b1 = ninf;
    int i1 = kNoExpert;
    for (int c = lane; c < E; c += 32) better(row[c], c, b1, i1);
    warp_argmax(b1, i1);
    T b2 = ninf;
    int i2 = kNoExpert;
    if (k == 2) {
      for (int c = lane; c < E; c += 32)
        if (c != i1) better(row[c], c, b2, i2);
      warp_argmax(b2, i2);
    }
    // max-shifted softmax over all E columns (gating.py:156-158)
    T m = b1;
    T sum = 0;
    for (int c = lane; c < E; c += 32) sum += exp_t(row[c] - m);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    if (probs != nullptr)
      for (int c = lane; c < E; c += 32) probs[t * E + c] = exp_t(row[c] - m) / sum;
    if (lane == 0) {
      ids[t * k] = i1;
      gate_probs[t * k] = exp_t(b1 - m) / sum;
      if (k == 2) {
        ids[t * k + 1] = i2;
        gate_probs[t * k + 1] = exp_t(b2 - m) / sum;
      }
    }
  }
}

// ============================================================ plan: tiles
// Block = one routing tile of 128 tokens, thread = token. local_rank[t, j] is
// the number of earlier assignments (token-major, gating.py:226) to the same
// expert inside the tile; tile_counts[tile, e] the tile's assignments to e.
MOE_DEV int warp_rank_same(int key, int my_lane) {
  unsigned m = __match_any_sync(0xffffffffu, key);
  return __popc(m & ((1u << my_lane) - 1u));
}

__global__ void plan_tiles_kernel(const int32_t* __restrict__ ids, int64_t S, int k, int E,
                                  int32_t* __restrict__ local_rank,
                                  int32_t* __restrict__ tile_counts) {
  extern __shared__ int cnt[];  // [4][E]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t t = tile * kRouteTile + tid;
  for (int i = tid; i < 4 * E; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const bool valid = t < S;
  // an id outside [0, E) matches no expert's indicator in the reference
  // (gating.py:229-230): it takes no slot and stays DROPPED
  int e0 = valid ? ids[t * k] : -1;
  int e1 = (valid && k == 2) ? ids[t * k + 1] : -2;
  const bool v0 = valid && e0 >= 0 && e0 < E;
  const bool v1 = valid && k == 2 && e1 >= 0 && e1 < E;
  if (!v0) e0 = -1;
  if (!v1) e1 = -2;
  int r0 = 0, r1 = 0;
  if (k == 1) {
    r0 = warp_rank_same(e0, lane);
  } else {
    for (int l = 0; l < 32; ++l) {
      int o0 = __shfl_sync(0xffffffffu, e0, l);
      int o1 = __shfl_sync(0xffffffffu, e1, l);
      if (l < lane) {
        r0 += (o0 == e0) + (o1 == e0);
        r1 += (o0 == e1) + (o1 == e1);
      }
    }
    r1 += (e0 == e1);  // a hand-built gate may repeat an expert: choice 0 comes first
  }
  if (v0) atomicAdd(&cnt[w * E + e0], 1);
  if (v1) atomicAdd(&cnt[w * E + e1], 1);
  __syncthreads();
  if (valid) {
    if (v0)
      for (int q = 0; q < w; ++q) r0 += cnt[q * E + e0];
    if (v1)
      for (int q = 0; q < w; ++q) r1 += cnt[q * E + e1];
    local_rank[t * k] = r0;
    if (k == 2) local_rank[t * k + 1] = r1;
  }
  for (int e = tid; e < E; e += blockDim.x)
    tile_counts[tile * E + e] = cnt[e] + cnt[E + e] + cnt[2 * E + e] + cnt[3 * E + e];
}

// ============================================================ plan: scan
// Block (32 experts x 32 chunks). tile_offsets[tile, e] = base[e] + sum of
// tile_counts[t' < tile, e]; totals[e] = sum over tiles; kept[e] = how many of
// this batch's assignments to e land below capacity given base[e].
__global__ void plan_scan_kernel(const int32_t* __restrict__ tile_counts, int64_t T, int E,
                                 int64_t cap, const int32_t* __restrict__ base,
                                 int32_t* __restrict__ tile_offsets, int32_t* __restrict__ totals,
                                 int32_t* __restrict__ kept) {
  __shared__ int part[32][33];
  pdl_trigger();
  pdl_wait();
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int e = blockIdx.x * 32 + tx;
  const int64_t chunk = (T + 31) / 32;
  const int64_t lo = ty * chunk, hi = min(T, lo + chunk);
  // chunk <= kReg (T <= 512 routing tiles = 65,536 tokens): the column's counts are
  // loaded once, all at the same time, and kept in registers for the second pass
  constexpr int kReg = 16;
  int v[kReg];
  const bool in_regs = chunk <= kReg;
  int s = 0;
  if (e < E) {
    if (in_regs) {
#pragma unroll
      for (int j = 0; j < kReg; ++j) v[j] = lo + j < hi ? tile_counts[(lo + j) * E + e] : 0;
#pragma unroll
      for (int j = 0; j < kReg; ++j) s += v[j];
    } else {
      for (int64_t i = lo; i < hi; ++i) s += tile_counts[i * E + e];
    }
  }
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0) {
    int run = (e < E && base != nullptr) ? base[e] : 0;
    const int b0 = run;
    for (int j = 0; j < 32; ++j) {
      int v = part[j][tx];
      part[j][tx] = run;
      run += v;
    }
    if (e < E) {
      const int total = run - b0;
      totals[e] = total;
      long long hi_kept = min((long long)run, (long long)cap);
      long long k_ = hi_kept - b0;
      kept[e] = (int)(k_ < 0 ? 0 : k_);
    }
  }
  __syncthreads();
  if (e < E) {
    int run = part[ty][tx];
    if (in_regs) {
#pragma unroll
      for (int j = 0; j < kReg; ++j) {
        if (lo + j < hi) tile_offsets[(lo + j) * E + e] = run;
        run += v[j];
      }
    } else {
      for (int64_t i = lo; i < hi; ++i) {
        tile_offsets[i * E + e] = run;
        run += tile_counts[i * E + e];
      }
    }
  }
}

// ============================================================ plan: slots
__global__ void plan_slots_kernel(const int32_t* __restrict__ ids,
                                  const int32_t* __restrict__ local_rank,
                                  const int32_t* __restrict__ tile_offsets, int64_t S, int k, int E,
                                  int64_t cap, int32_t* __restrict__ slots) {
  const int64_t n = S * k;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = a / k;
    const int e = ids[a];
    if (e < 0 || e >= E) {  // matches no expert (plan_tiles_kernel)
      slots[a] = -1;
      continue;
    }
    const int64_t slot = (int64_t)tile_offsets[(t / kRouteTile) * E + e] + local_rank[a];
    slots[a] = slot < cap ? (int32_t)slot : -1;
  }
}

// ============================================================ int64 scan
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanBlock = kScanThreads * kScanItems;

template <bool kWriteOut>
__global__ void scan_i64_block_kernel(const int64_t* __restrict__ in, int64_t n,
                                      const int64_t* __restrict__ block_base,
                                      int64_t* __restrict__ out, int64_t* __restrict__ block_sums) {
  __shared__ int64_t warp_tot[kScanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanBlock + (int64_t)tid * kScanItems;
  int64_t v[kScanItems];
  int64_t run = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = base + i;
    v[i] = idx < n ? in[idx] : 0;
    const int64_t x = v[i];
    v[i] = run;  // exclusive within thread
    run += x;
  }
  // warp inclusive scan of per-thread totals
  int64_t incl = run;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int64_t o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int64_t wt = lane < kScanThreads / 32 ? warp_tot[lane] : 0;
    int64_t wi = wt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int64_t o = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += o;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = wi - wt;  // exclusive warp offsets
    if (lane == kScanThreads / 32 - 1 && block_sums != nullptr) block_sums[blockIdx.x] = wi;
  }
  __syncthreads();
  if (kWriteOut) {
    const int64_t off = (incl - run) + warp_tot[w] + (block_base ? block_base[blockIdx.x] : 0);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const int64_t idx = base + i;
      if (idx < n) out[idx] = v[i] + off;
    }
  }
}

// ============================================================ Blelloch f64
// One tree level of gating.py:189-201, applied with the same pairings so the
// float result matches NumPy bit for bit (plain IEEE adds, no contraction).
__global__ void blelloch_up_kernel(double* tree, int64_t m, int64_t d) {
  const int64_t pairs = m / (2 * d);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pairs;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (2 * i + 2) * d - 1, l = (2 * i + 1) * d - 1;
    tree[r] = __dadd_rn(tree[r], tree[l]);
  }
}

__global__ void blelloch_down_kernel(double* tree, int64_t m, int64_t d) {
  const int64_t pairs = m / (2 * d);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pairs;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (2 * i + 2) * d - 1, l = (2 * i + 1) * d - 1;
    const double left = tree[l];
    tree[l] = tree[r];
    tree[r] = __dadd_rn(tree[r], left);
  }
}

// ============================================================ scatter
// Warp per token: the row is read once and stored to each kept (expert, slot)
// of the token. With local_rank/tile_offsets given, the slot is resolved here
// (and written to slots) - the layer path fuses plan_slots into dispatch.
// For the k=1 fused-combine layer path it also records, per expert-buffer row,
// the source token and its gate probability (read by the GEMM2 epilogue), and
// writes out[t] = x[t] for tokens whose every assignment was dropped
// (arch.py:389: dropped tokens ride the skip connection).
// TPW tokens per warp (32/TPW lanes each), as in combine_kernel.
template <typename V, int TPW = 1>
__global__ void scatter_kernel(ScatterArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int LPT = 32 / TPW;  // lanes per token
  const int lane = threadIdx.x & (LPT - 1);
  const int64_t slots_total = (int64_t)gridDim.x * (blockDim.x >> 5) * TPW;
  const int64_t nvec = a.row_bytes / (int64_t)sizeof(V);
  const int k = a.k;
  for (int64_t t = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * TPW +
                   (threadIdx.x & 31) / LPT;
       t < a.S; t += slots_total) {
    int64_t dst0 = -1, dst1 = -1;
    uint8_t* base0 = a.buf;
    uint8_t* base1 = a.buf;
    for (int j = 0; j < k; ++j) {
      const int e = a.ids[t * k + j];
      int64_t slot;
      if (a.local_rank != nullptr) {
        slot = (int64_t)a.tile_offsets[(t / kRouteTile) * a.E + e] + a.local_rank[t * k + j];
        if (slot >= a.cap) slot = -1;
        if (lane == 0) a.slots[t * k + j] = (int32_t)slot;
      } else {
        slot = a.slots[t * k + j];
      }
      int64_t d = -1;
      if (slot >= 0) {
        // expert-buffer row e*cap + slot, or (EP send buffer) row_base[e] + slot - slot_base[e]
        d = a.row_base != nullptr
                ? (int64_t)a.row_base[e] + slot - (a.slot_base ? a.slot_base[e] : 0)
                : (int64_t)e * a.cap + slot;
        uint8_t* base = a.buf;
        int32_t* rtok = a.row_token;
        float* rprob = a.row_prob;
        int32_t* rsrc = nullptr;
        if (a.peer_buf != nullptr) {  // EP over NVLink: the owner rank's receive buffer
          const int owner = e / a.e_per_rank;
          base = a.peer_buf[owner];
          rtok = a.peer_token[owner];
          rprob = a.peer_prob[owner];
          if (a.peer_src != nullptr) rsrc = a.peer_src[owner];
        }
        if (j == 0) { dst0 = d; base0 = base; } else { dst1 = d; base1 = base; }
        if (lane == 0) {
          if (a.occupied != nullptr) a.occupied[d] = 1;
          if (rtok != nullptr) {
            // push return: where the owner sends the row back (source rank, row t*k+j)
            rtok[d] = rsrc != nullptr ? (int32_t)(t * k + j) : (int32_t)t;
            rprob[d] = a.gate_probs[t * k + j];
            if (rsrc != nullptr) rsrc[d] = a.my_rank;
          }
        }
      }
      if (a.row_index != nullptr && lane == 0)
        a.row_index[t * k + j] = (a.peer_src != nullptr && d >= 0) ? (int32_t)(t * k + j) : (int32_t)d;
    }
    V* d0 = nullptr;
    V* d1 = nullptr;
    if (dst0 >= 0 || dst1 >= 0) {
      // route-only mode (no expert buffer): the grouped GEMM gathers the row itself
      if (a.buf == nullptr && a.peer_buf == nullptr) continue;
      d0 = dst0 >= 0 ? reinterpret_cast<V*>(base0 + dst0 * a.row_bytes) : nullptr;
      d1 = dst1 >= 0 ? reinterpret_cast<V*>(base1 + dst1 * a.row_bytes) : nullptr;
    } else {
      if (a.out_dropped == nullptr) continue;
      d0 = reinterpret_cast<V*>(a.out_dropped + t * a.row_bytes);  // out = x
    }
    const V* src = reinterpret_cast<const V*>(a.x + t * a.row_bytes);
    constexpr int U = 4;
    int64_t i = lane;
    for (; i + LPT * (U - 1) < nvec; i += LPT * U) {
      V r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = __ldg(src + i + LPT * u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (d0) d0[i + LPT * u] = r[u];
        if (d1) d1[i + LPT * u] = r[u];
      }
    }
    for (; i < nvec; i += LPT) {
      V r = __ldg(src + i);
      if (d0) d0[i] = r;
      if (d1) d1[i] = r;
    }
  }
  // peer stores must be performed (acknowledged) before the barrier kernel signals
  if (a.peer_buf != nullptr) __threadfence_system();
}

// ============================================================ combine
template <typename T>
struct Acc {
  using type = float;
};
template <>
struct Acc<double> {
  using type = double;
};

MOE_DEV float to_acc(float v) { return v; }
MOE_DEV float to_acc(__nv_bfloat16 v) { return __bfloat162float(v); }
MOE_DEV double to_acc(double v) { return v; }
template <typename T>
MOE_DEV T from_acc(float v);
template <>
MOE_DEV float from_acc<float>(float v) {
  return v;
}
template <>
MOE_DEV __nv_bfloat16 from_acc<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
MOE_DEV double from_acc_d(double v) { return v; }

MOE_DEV float add_rn(float a, float b) { return __fadd_rn(a, b); }
MOE_DEV double add_rn(double a, double b) { return __dadd_rn(a, b); }
MOE_DEV float mul_rn(float a, float b) { return __fmul_rn(a, b); }
MOE_DEV double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// out[t] = (x[t] + sum_j p_j * y[row_j]) + shared[t]   (arch.py:389-391, :406-410)
// kExpertOrder: contributions summed in ascending expert id (forward_layer's
// loop over experts); otherwise in choice order (combine_tokens' np.add.at).
// Every multiply/add is individually rounded so f64 results match NumPy.
// Warp per token; each lane moves VEC elements (16 B) per access.
template <typename T, int VEC>
struct alignas(sizeof(T) * VEC) Pack {
  T v[VEC];
};

// TPW tokens per warp (32/TPW lanes each): TPW = 2 halves the warps, so 16K
// tokens fill ~1.7 waves of resident warps instead of ~3.5, while every warp
// keeps two independent index -> row load chains in flight.
template <typename T, typename P, bool kExpertOrder, int VEC, int TPW = 1>
__global__ void combine_kernel(const T* __restrict__ y, int64_t S, int M, int k, int E, int64_t cap,
                               const int32_t* __restrict__ ids, const int32_t* __restrict__ slots,
                               const int32_t* __restrict__ row_index, const P* __restrict__ gp,
                               const T* __restrict__ x, const T* __restrict__ shared,
                               T* __restrict__ out) {
  using A = typename Acc<T>::type;
  using V = Pack<T, VEC>;
  constexpr int LPT = 32 / TPW;  // lanes per token
  const int lane = threadIdx.x & (LPT - 1);
  const int64_t slots_total = (int64_t)gridDim.x * (blockDim.x >> 5) * TPW;
  const int nv = M / VEC;
  for (int64_t t = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * TPW +
                   (threadIdx.x & 31) / LPT;
       t < S; t += slots_total) {
    int64_t r0 = -1, r1 = -1;
    A p0 = 0, p1 = 0;
    int e0 = 0, e1 = 0, n = 0;
    for (int j = 0; j < k; ++j) {
      int64_t r;
      if (row_index != nullptr) {
        r = row_index[t * k + j];
      } else {
        const int s = slots[t * k + j];
        r = s >= 0 ? (int64_t)ids[t * k + j] * cap + s : -1;
      }
      if (r >= 0) {
        const A pj = (A)gp[t * k + j];
        const int ej = ids[t * k + j];
        if (n == 0) { r0 = r; p0 = pj; e0 = ej; }
        else { r1 = r; p1 = pj; e1 = ej; }
        ++n;
      }
    }
    if (kExpertOrder && n == 2 && e1 < e0) {
      int64_t tr = r0; r0 = r1; r1 = tr;
      A tp = p0; p0 = p1; p1 = tp;
    }
    const V* y0 = reinterpret_cast<const V*>(y + (n > 0 ? r0 : 0) * M);
    const V* y1 = reinterpret_cast<const V*>(y + (n > 1 ? r1 : 0) * M);
    const V* xv = reinterpret_cast<const V*>(x + t * M);
    const V* sv = reinterpret_cast<const V*>(shared + t * M);
    V* ov = reinterpret_cast<V*>(out + t * M);
#pragma unroll 4
    for (int c = lane; c < nv; c += LPT) {
      V a0, a1, xa, sa;
      if (n > 0) a0 = y0[c];
      if (n > 1) a1 = y1[c];
      if (x != nullptr) xa = xv[c];
      if (shared != nullptr) sa = sv[c];
      V o;
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        A acc = 0;  // the zero accumulator of scatter_rows / np.add.at
        if (n > 0) acc = add_rn(acc, mul_rn(p0, to_acc(a0.v[i])));
        if (n > 1) acc = add_rn(acc, mul_rn(p1, to_acc(a1.v[i])));
        A r = acc;
        if (x != nullptr) r = add_rn(to_acc(xa.v[i]), acc);
        if (shared != nullptr) r = add_rn(r, to_acc(sa.v[i]));
        if constexpr (sizeof(T) == 8) {
          o.v[i] = r;
        } else {
          o.v[i] = from_acc<T>(r);
        }
      }
      ov[c] = o;
    }
  }
}

// Block-staged combine (16-B vector path): a block owns TB consecutive tokens.
// Its first TB threads resolve the tokens' routing (ids / slots / row_index / gp
// -> up to two (row, prob) pairs in summation order) into shared memory in one
// coalesced pass, so combine_kernel's per-token index -> row -> data chain
// collapses into one round trip per block; then each warp streams whole rows,
// all U 16-B loads of every input row issued before any is consumed. Same
// arithmetic in the same order as combine_kernel.
template <typename T>
struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
  MOE_DEV static void unpack(const uint4& u, typename Acc<T>::type (&v)[N]) {
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = to_acc(e[i]);
  }
  MOE_DEV static uint4 pack(const typename Acc<T>::type (&v)[N]) {
    uint4 u;
    T* e = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if constexpr (sizeof(T) == 8) {
        e[i] = v[i];
      } else {
        e[i] = from_acc<T>(v[i]);
      }
    }
    return u;
  }
};

template <typename T, typename P, bool kExpertOrder, int TB, int U, bool kShared>
__global__ void __launch_bounds__(256, 3) combine_tb_kernel(
    const T* __restrict__ y, int64_t S, int M, int k, int E, int64_t cap,
    const int32_t* __restrict__ ids, const int32_t* __restrict__ slots,
    const int32_t* __restrict__ row_index, const P* __restrict__ gp, const T* __restrict__ x,
    const T* __restrict__ shared, T* __restrict__ out) {
  using A = typename Acc<T>::type;
  using W = Vec16<T>;
  constexpr int NV = W::N;
  __shared__ int64_t s_r[2][TB];
  __shared__ A s_p[2][TB];
  __shared__ int s_n[TB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nv = M / NV;  // 16-B vectors per row
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  pdl_trigger();
  pdl_wait();
  // persistent grid (resident blocks only): block b owns the contiguous token range
  // [b*S/grid, (b+1)*S/grid), so the work is balanced to a token, not to a batch
  const int64_t lo = (int64_t)blockIdx.x * S / gridDim.x;
  const int64_t hi = (int64_t)(blockIdx.x + 1) * S / gridDim.x;
  for (int64_t t0 = lo; t0 < hi; t0 += TB) {
    if (threadIdx.x < TB && t0 + threadIdx.x < hi) {
      const int64_t t = t0 + threadIdx.x;
      int64_t r0 = -1, r1 = -1;
      A p0 = 0, p1 = 0;
      int e0 = 0, e1 = 0, n = 0;
      for (int j = 0; j < k; ++j) {
        int64_t r;
        if (row_index != nullptr) {
          r = row_index[t * k + j];
        } else {
          const int sl = slots[t * k + j];
          r = sl >= 0 ? (int64_t)ids[t * k + j] * cap + sl : -1;
        }
        if (r >= 0) {
          const A pj = (A)gp[t * k + j];
          const int ej = ids[t * k + j];
          if (n == 0) { r0 = r; p0 = pj; e0 = ej; }
          else { r1 = r; p1 = pj; e1 = ej; }
          ++n;
        }
      }
      if (kExpertOrder && n == 2 && e1 < e0) {
        int64_t tr = r0; r0 = r1; r1 = tr;
        A tp = p0; p0 = p1; p1 = tp;
      }
      s_r[0][threadIdx.x] = r0;
      s_r[1][threadIdx.x] = r1;
      s_p[0][threadIdx.x] = p0;
      s_p[1][threadIdx.x] = p1;
      s_n[threadIdx.x] = n;
    }
    __syncthreads();
    for (int i = warp; i < TB && t0 + i < hi; i += nw) {
      const int64_t t = t0 + i;
      const int n = s_n[i];
      const A p0 = s_p[0][i], p1 = s_p[1][i];
      const uint4* y0 = reinterpret_cast<const uint4*>(y + (n > 0 ? s_r[0][i] : 0) * M);
      const uint4* y1 = reinterpret_cast<const uint4*>(y + (n > 1 ? s_r[1][i] : 0) * M);
      const uint4* xv = reinterpret_cast<const uint4*>(x + t * M);
      const uint4* sv = reinterpret_cast<const uint4*>(shared + t * M);
      uint4* ov = reinterpret_cast<uint4*>(out + t * M);
      for (int c0 = 0; c0 < nv; c0 += 32 * U) {
        uint4 a0[U], a1[U], xa[U], sa[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * 32 + lane;
          const bool in = c < nv;
          a0[u] = (in && n > 0) ? __ldcs(y0 + c) : z;
          a1[u] = (in && n > 1) ? __ldcs(y1 + c) : z;
          xa[u] = (in && x != nullptr) ? __ldcs(xv + c) : z;
          if constexpr (kShared) sa[u] = in ? __ldcs(sv + c) : z;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c >= nv) continue;
          A v0[NV], v1[NV], vx[NV], vs[NV], o[NV];
          W::unpack(a0[u], v0);
          W::unpack(a1[u], v1);
          W::unpack(xa[u], vx);
          if constexpr (kShared) W::unpack(sa[u], vs);
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            A acc = 0;  // the zero accumulator of scatter_rows / np.add.at
            if (n > 0) acc = add_rn(acc, mul_rn(p0, v0[q]));
            if (n > 1) acc = add_rn(acc, mul_rn(p1, v1[q]));
            A r = acc;
            if (x != nullptr) r = add_rn(vx[q], acc);
            if constexpr (kShared) r = add_rn(r, vs[q]);
            o[q] = r;
          }
          __stcs(ov + c, W::pack(o));
        }
      }
    }
    __syncthreads();
  }
}

// ============================================================ load-balance loss
// E * sum_e (count_e / (S k)) * (mean_t probs[t, e]) with pre-drop counts
// (arch.py:297-313). Statistics in float64.
template <typename T>
__global__ void aux_stats_kernel(const int32_t* __restrict__ ids, int64_t S, int k, int E,
                                 const T* __restrict__ probs, double* __restrict__ ws) {
  const int64_t rows_per = (S + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(S, r0 + rows_per);
  for (int c = threadIdx.x; c < E; c += blockDim.x) {
    double acc = 0.0;
    for (int64_t r = r0; r < r1; ++r) acc += (double)probs[r * E + c];
    if (r1 > r0) atomicAdd(&ws[c], acc);
  }
  for (int64_t a = r0 * k + threadIdx.x; a < r1 * k; a += blockDim.x) {
    const int e = ids[a];
    if (e >= 0 && e < E) atomicAdd(&ws[E + e], 1.0);  // the host rejects others first
  }
}

__global__ void aux_finalize_kernel(int64_t S, int k, int E, const double* __restrict__ ws,
                                    const int32_t* __restrict__ counts,
                                    const float* __restrict__ probsum, double* out) {
  __shared__ double part[32];
  double acc = 0.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const double cnt = counts ? (double)counts[e] : ws[E + e];
    const double ps = probsum ? (double)probsum[e] : ws[e];
    acc += (cnt / ((double)S * k)) * (ps / (double)S);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    out[0] = S > 0 ? (double)E * t : 0.0;
  }
}

int launch_aux_loss(const int32_t* ids, int64_t S, int k, int E, const void* probs, int dtype,
                    const int32_t* counts, const float* probsum, double* out, double* ws,
                    cudaStream_t st) {
  if (counts == nullptr || probsum == nullptr) {
    cudaMemsetAsync(ws, 0, 2 * (size_t)E * sizeof(double), st);
    if (S > 0) {
      const int g = (int)(S < 148 * 4 ? S : 148 * 4);
      if (dtype == MOE_F64)
        aux_stats_kernel<double><<<g, 256, 0, st>>>(ids, S, k, E, (const double*)probs, ws);
      else if (dtype == MOE_F32)
        aux_stats_kernel<float><<<g, 256, 0, st>>>(ids, S, k, E, (const float*)probs, ws);
      else
        return MOE_EINVAL;
    }
  }
  aux_finalize_kernel<<<1, 256, 0, st>>>(S, k, E, ws, counts, probsum, out);
  return (int)cudaGetLastError();
}

// ============================================================ launchers
static int grid_for(int64_t work, int per_block, int cap_blocks = 148 * 32) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap_blocks) g = cap_blocks;
  return (int)g;
}

int launch_topk_gate(const void* logits, int dtype, int64_t S, int E, int k, int32_t* ids,
                     void* gate_probs, void* probs, cudaStream_t st) {
  if (S == 0) return 0;
  const int threads = 256;
  const int g = grid_for(S, threads / 32, 148 * 64);
  if (dtype == MOE_F32)
    topk_gate_kernel<float><<<g, threads, 0, st>>>((const float*)logits, S, E, k, ids,
                                                   (float*)gate_probs, (float*)probs);
  else if (dtype == MOE_F64)
    topk_gate_kernel<double><<<g, threads, 0, st>>>((const double*)logits, S, E, k, ids,
                                                    (double*)gate_probs, (double*)probs);
  else
    return MOE_EINVAL;
  return (int)cudaGetLastError();
}

int launch_plan(const int32_t* ids, int64_t S, int k, int E, int64_t cap, const int32_t* base,
                int32_t* local_rank, int32_t* tile_counts, int32_t* tile_offsets, int32_t* totals,
                int32_t* kept, int32_t* slots, bool tiles, bool scan, bool do_slots,
                cudaStream_t st) {
  const int64_t T = (S + kRouteTile - 1) / kRouteTile;
  if (tiles && T > 0) {
    plan_tiles_kernel<<<(unsigned)T, kRouteTile, 4 * E * sizeof(int), st>>>(ids, S, k, E,
                                                                           local_rank, tile_counts);
  }
  if (scan) {
    dim3 blk(32, 32);
    launch_pdl(plan_scan_kernel, dim3((E + 31) / 32), blk, 0, st, tile_counts, T, E, cap, base, tile_offsets,
                                                    totals, kept);
  }
  if (do_slots && S > 0) {
    plan_slots_kernel<<<grid_for(S * k, 256), 256, 0, st>>>(ids, local_rank, tile_offsets, S, k, E,
                                                            cap, slots);
  }
  return (int)cudaGetLastError();
}

int64_t scan_i64_workspace_elems(int64_t n) {
  int64_t total = 0;
  while (n > kScanBlock) {
    n = (n + kScanBlock - 1) / kScanBlock;
    total += 2 * n;
  }
  return total + 1;
}

static void scan_i64_rec(const int64_t* in, int64_t n, int64_t* out, int64_t* ws,
                         cudaStream_t st) {
  const int64_t blocks = (n + kScanBlock - 1) / kScanBlock;
  if (blocks <= 1) {
    scan_i64_block_kernel<true><<<1, kScanThreads, 0, st>>>(in, n, nullptr, out, nullptr);
    return;
  }
  int64_t* sums = ws;
  int64_t* sums_scan = ws + blocks;
  scan_i64_block_kernel<false><<<(unsigned)blocks, kScanThreads, 0, st>>>(in, n, nullptr, nullptr,
                                                                          sums);
  scan_i64_rec(sums, blocks, sums_scan, ws + 2 * blocks, st);
  scan_i64_block_kernel<true><<<(unsigned)blocks, kScanThreads, 0, st>>>(in, n, sums_scan, out,
                                                                         nullptr);
}

int launch_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* ws, cudaStream_t st) {
  if (n == 0) return 0;
  scan_i64_rec(in, n, out, ws, st);
  return (int)cudaGetLastError();
}

int launch_blelloch_f64(double* tree, int64_t m, cudaStream_t st) {
  // tree holds the zero-padded input (m a power of two); exclusive scan in place
  for (int64_t d = 1; d < m; d <<= 1)
    blelloch_up_kernel<<<grid_for(m / (2 * d), 256), 256, 0, st>>>(tree, m, d);
  cudaMemsetAsync(tree + (m - 1), 0, sizeof(double), st);
  for (int64_t d = m >> 1; d >= 1; d >>= 1)
    blelloch_down_kernel<<<grid_for(m / (2 * d), 256), 256, 0, st>>>(tree, m, d);
  return (int)cudaGetLastError();
}

int launch_scatter(const ScatterArgs& args, cudaStream_t st) {
  if (args.S == 0) return 0;
  const int threads = 256;
  int g = grid_for(args.S, threads / 32, 148 * 64);
  if (comm_block_limit() > 0 && g > comm_block_limit()) g = comm_block_limit();
  // several tokens per warp (more independent rows in flight per warp): two for
  // the local dispatch (101 -> 91 us at C3), four for stores over NVLink (N=2:
  // 0.33 -> 0.28 -> 0.24 ms)
  static const int tpw_env = [] {
    const char* v = getenv("MOE_SCATTER_TPW");
    return v ? atoi(v) : 0;
  }();
  const int tpw = tpw_env ? tpw_env : (args.peer_buf != nullptr ? 4 : 2);
  if (tpw == 4 && args.row_bytes % 16 == 0) {
    const int g4 = (g + 3) / 4;
    return (int)launch_pdl(scatter_kernel<uint4, 4>, dim3(g4 > 0 ? g4 : 1), dim3(threads), 0, st,
                           args);
  } else if (tpw == 2 && args.row_bytes % 16 == 0) {
    const int g2 = (g + 1) / 2;
    return (int)launch_pdl(scatter_kernel<uint4, 2>, dim3(g2 > 0 ? g2 : 1), dim3(threads), 0, st,
                           args);
  } else if (args.row_bytes % 16 == 0)
    scatter_kernel<uint4><<<g, threads, 0, st>>>(args);
  else if (args.row_bytes % 8 == 0)
    scatter_kernel<uint2><<<g, threads, 0, st>>>(args);
  else if (args.row_bytes % 4 == 0)
    scatter_kernel<uint32_t><<<g, threads, 0, st>>>(args);
  else
    scatter_kernel<uint16_t><<<g, threads, 0, st>>>(args);
  return (int)cudaGetLastError();
}

// Resident blocks of a kernel on the current device (persistent grids), cached
// per (kernel instance, device ordinal).
template <typename Kern>
static int64_t resident_blocks(Kern kern, int threads) {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    int per_sm = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
      sms = 148;
    v = per_sm * sms;
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

template <typename T, typename P, int VEC>
static void combine_vec(bool expert_order, int g, int threads, cudaStream_t st, const void* y,
                        int64_t S, int M, int k, int E, int64_t cap, const int32_t* ids,
                        const int32_t* slots, const int32_t* row_index, const void* gp,
                        const void* x, const void* shared, void* out) {
  static const int tpw = [] {
    const char* v = getenv("MOE_COMBINE_TPW");
    return v ? atoi(v) : 0;
  }();
  // default (MOE_COMBINE_TPW unset / 0): the block-staged kernel, 32 tokens per
  // 256-thread block; MOE_COMBINE_TB=16 halves the block's token batch
  static const int tb = [] {
    const char* v = getenv("MOE_COMBINE_TB");
    return v ? atoi(v) : 32;
  }();
  if (tpw == 0 && VEC > 1) {
    const int64_t blocks = (S + tb - 1) / tb;
#define MOE_COMBINE_TB(TB_, EO_, SH_)                                                           \
  {                                                                                             \
    auto kern = combine_tb_kernel<T, P, EO_, TB_, (sizeof(T) == 2 ? 2 : 4), SH_>;               \
    const int64_t res = resident_blocks(kern, 256);                                             \
    const int gb = (int)(blocks < res ? blocks : res);                                          \
    launch_pdl(kern, dim3(gb), dim3(256), 0, st, (const T*)y, S, M, k, E, cap, ids, slots,      \
               row_index, (const P*)gp, (const T*)x, (const T*)shared, (T*)out);               \
  }
    const bool sh = shared != nullptr;
    if (tb == 16) {
      if (expert_order) {
        if (sh) MOE_COMBINE_TB(16, true, true) else MOE_COMBINE_TB(16, true, false)
      } else {
        if (sh) MOE_COMBINE_TB(16, false, true) else MOE_COMBINE_TB(16, false, false)
      }
    } else {
      if (expert_order) {
        if (sh) MOE_COMBINE_TB(32, true, true) else MOE_COMBINE_TB(32, true, false)
      } else {
        if (sh) MOE_COMBINE_TB(32, false, true) else MOE_COMBINE_TB(32, false, false)
      }
    }
#undef MOE_COMBINE_TB
    return;
  }
  if (tpw == 4 && VEC > 1) {
    const int g4 = (g + 3) / 4;
    if (expert_order)
      combine_kernel<T, P, true, VEC, 4><<<g4, threads, 0, st>>>(
          (const T*)y, S, M, k, E, cap, ids, slots, row_index, (const P*)gp, (const T*)x,
          (const T*)shared, (T*)out);
    else
      combine_kernel<T, P, false, VEC, 4><<<g4, threads, 0, st>>>(
          (const T*)y, S, M, k, E, cap, ids, slots, row_index, (const P*)gp, (const T*)x,
          (const T*)shared, (T*)out);
    return;
  }
  if (tpw == 2 && VEC > 1) {
    const int g2 = (g + 1) / 2;
    if (expert_order)
      combine_kernel<T, P, true, VEC, 2><<<g2, threads, 0, st>>>(
          (const T*)y, S, M, k, E, cap, ids, slots, row_index, (const P*)gp, (const T*)x,
          (const T*)shared, (T*)out);
    else
      combine_kernel<T, P, false, VEC, 2><<<g2, threads, 0, st>>>(
          (const T*)y, S, M, k, E, cap, ids, slots, row_index, (const P*)gp, (const T*)x,
          (const T*)shared, (T*)out);
    return;
  }
  if (expert_order)
    combine_kernel<T, P, true, VEC><<<g, threads, 0, st>>>(
        (const T*)y, S, M, k, E, cap, ids, slots, row_index, (const P*)gp, (const T*)x,
        (const T*)shared, (T*)out);
  else
    combine_kernel<T, P, false, VEC><<<g, threads, 0, st>>>(
        (const T*)y, S, M, k, E, cap, ids, slots, row_index, (const P*)gp, (const T*)x,
        (const T*)shared, (T*)out);
}

template <typename T, typename P>
static void combine_dispatch(bool expert_order, int g, int threads, cudaStream_t st, const void* y,
                             int64_t S, int M, int k, int E, int64_t cap, const int32_t* ids,
                             const int32_t* slots, const int32_t* row_index, const void* gp,
                             const void* x, const void* shared, void* out) {
  constexpr int VEC = 16 / sizeof(T);
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; };
  const bool vec_ok = (M % VEC) == 0 && aligned(out) && (y == nullptr || aligned(y)) &&
                      (x == nullptr || aligned(x)) && (shared == nullptr || aligned(shared));
  if (vec_ok)
    combine_vec<T, P, VEC>(expert_order, g, threads, st, y, S, M, k, E, cap, ids, slots, row_index,
                           gp, x, shared, out);
  else
    combine_vec<T, P, 1>(expert_order, g, threads, st, y, S, M, k, E, cap, ids, slots, row_index,
                         gp, x, shared, out);
}

int launch_combine(const void* y, int dtype, int64_t S, int M, int k, int E, int64_t cap,
                   const int32_t* ids, const int32_t* slots, const int32_t* row_index,
                   const void* gate_probs, int gp_dtype, const void* x, const void* shared,
                   void* out, int expert_order, cudaStream_t st) {
  if (S == 0) return 0;
  const int threads = 256;
  const int g = grid_for(S, threads / 32, 148 * 64);
  if (dtype == MOE_F64 && gp_dtype == MOE_F64)
    combine_dispatch<double, double>(expert_order, g, threads, st, y, S, M, k, E, cap, ids, slots,
                                     row_index, gate_probs, x, shared, out);
  else if (dtype == MOE_F32 && gp_dtype == MOE_F32)
    combine_dispatch<float, float>(expert_order, g, threads, st, y, S, M, k, E, cap, ids, slots,
                                   row_index, gate_probs, x, shared, out);
  else if (dtype == MOE_BF16 && gp_dtype == MOE_F32)
    combine_dispatch<__nv_bfloat16, float>(expert_order, g, threads, st, y, S, M, k, E, cap, ids,
                                           slots, row_index, gate_probs, x, shared, out);
  else
    return MOE_EINVAL;
  return (int)cudaGetLastError();
}

}  // namespace moe
