// tcgen05 + TMA grouped GEMM for sm_100a (bf16 in, fp32 accumulate in TMEM).
//
//   D[rows of group g] = epilogue( A[rows of g] (r x K) . B_w(g)^T (K x N) )
//
// Used for
//   * the expert FFN halves of forward_ffn (arch.py:368-369): GEMM1 with a
//     bias + tanh-GELU epilogue, GEMM2 with a bias epilogue, one group per
//     expert (or per (source rank, expert) segment under expert parallelism);
//   * the gate GEMM (arch.py:384) with a fused routing epilogue: softmax over
//     all E logits, top-k with lower-index ties (gating.py:142-163) and the
//     per-tile capacity ranks that build_dispatch_plan scans (gating.py:211-247).
//
// Persistent kernel, one CTA per SM, 6 warps:
//   warp 0    TMA producer (A and B tiles, 128B swizzle, STAGES-deep ring)
//   warp 1    TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2-5 epilogue: tcgen05.ld (32 lanes x 32 columns) -> registers -> HBM
// The fp32 accumulator is double buffered in TMEM (2 x BN columns) so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#include "common.cuh"
#include <type_traits>

#include "moe_kernels.h"

#include <cudaTypedefs.h>

#include <cstdlib>
#include <atomic>
#include <mutex>

namespace moe {

// EPI_BIAS_COMBINE (GEMM2 of a k=1 layer): out[token(row)] = x[token] + p(row) * (acc + b2),
// i.e. combine_tokens + the residual add of arch.py:389 fused into the epilogue.
// Training epilogues (layer backward):
//   EPI_GELU_SAVE: as EPI_BIAS_GELU, also storing the pre-activation a = acc + b1 to `out`
//   EPI_GELU_BWD : D = acc * gelu'(a), a read from `x_resid` at the same row (dA = dH * gelu'(a))
// Weight-gradient mode (both operands MN-major, K = token rows of the group):
//   EPI_WGRAD    : D[g] (P x N, bf16) = X_g^T Y_g, X_g / Y_g the first k_rows[g] rows
//                  of group g (rows [g*k_stride, +k_rows[g]) of X and Y)
//   EPI_WGRAD_ACC: Dacc (P x N, fp32) += X_g^T Y_g for every g (split-K over groups)
// Residual-MoE layer (arch.py:389-391) as ONE launch per GEMM: the shared MLP runs
// as extra groups of the expert launches (its tokens split into row_stride-row
// groups, weight index E):
//   GEMM1: groups >= a2_group read their A rows from a second matrix (map_a2 = x)
//   EPI_BIAS_RESID (GEMM2): groups < rc_group are experts, D = acc + b2 (the expert
//     outputs y); groups >= rc_group are the shared MLP, whose epilogue waits until
//     every expert tile has stored (device counter) and emits
//     out[t] = (x[t] + sum_j p_j y[e_j*cap + slot_j]) + (acc + b2_shared).
// MOE_GATE_TRACE (debug builds only, tools/gate_trace.sh): %globaltimer stamps of
// the gate's phases in CTA 0, read back with moe_debug_gate_trace()
#ifdef MOE_GATE_TRACE
__device__ unsigned long long g_gate_trace[16];
#define GATE_TRACE(i)                                                              \
  do {                                                                             \
    if (EPI == EPI_GATE && blockIdx.x == 0) {                                      \
      unsigned long long t_;                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                       \
      g_gate_trace[i] = t_;                                                        \
    }                                                                              \
  } while (0)
#else
#define GATE_TRACE(i) \
  do {                \
  } while (0)
#endif

enum { EPI_BIAS = 0, EPI_BIAS_GELU = 1, EPI_GATE = 2, EPI_BIAS_COMBINE = 3, EPI_GELU_SAVE = 4,
       EPI_GELU_BWD = 5, EPI_WGRAD = 6, EPI_WGRAD_ACC = 7, EPI_BIAS_RESID = 8,
       EPI_COMBINE_PUSH = 9 };
// EPI_COMBINE_PUSH: EPI_BIAS_COMBINE for the EP push return (rows stored to the
// sources over NVLink through the coalescing smem stage); its own instance so the
// single-GPU fused-combine GEMM keeps its registers
template <int EPI>
constexpr bool is_combine() {
  return EPI == EPI_BIAS_COMBINE || EPI == EPI_COMBINE_PUSH;
}

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
// warps 0-1: TMA producer, MMA issuer; then the epilogue warps. The expert
// GEMMs use 8 epilogue warps (2 per TMEM lane quarter, each owning half of the
// tile's columns) so two warps per scheduler hide the epilogue's latencies;
// the gate epilogue (thread = token, full row of logits) uses 4.
// (+1 fix-up warp in the weight-gradient modes: see the partial K block)
template <int EW, int EPI = EPI_BIAS>
constexpr int threads_for() {
  return 64 + 32 * EW + ((EPI == EPI_WGRAD || EPI == EPI_WGRAD_ACC) ? 32 : 0);
}
constexpr int kMaxGroups = 2048;
constexpr int kTileQ = 8;  // dynamic tile scheduler: queue depth (producer runs <= ~3 tiles ahead)

struct GemmArgs {
  const float* bias;          // [num_weights, N] fp32 (may be null)
  __nv_bfloat16* D;           // [a_rows, N]
  int K, N;
  int G;                      // groups
  const int32_t* row_start;   // [G] or null -> g * row_stride
  int64_t row_stride;
  const int32_t* rows;        // [G] device rows per group (or null -> rows_const)
  int64_t rows_const;
  const int32_t* weight_idx;  // [G] or null -> g
  // gate epilogue
  int E, k;
  int64_t S;
  float* logits;              // [S, E] optional
  int32_t* ids;               // [S, k]
  float* gate_probs;          // [S, k]
  int32_t* local_rank;        // [S, k]
  int32_t* tile_counts;       // [T, E]
  float* probsum;             // [E] optional: column sums of the softmax (load-balance loss)
  // fused combine epilogue
  const int32_t* row_token;   // [a_rows] token of each expert-buffer row
  const float* row_prob;      // [a_rows] its gate probability
  const __nv_bfloat16* x_resid;  // [S, N] indexed by token, or [a_rows, N] by row (x_by_row)
  __nv_bfloat16* out;            // [S, N]
  // EP owner side: the residual x is the (dispatched) row itself and the combined
  // row is stored at the same row of `out` (receive layout); the source rank then
  // pulls it over NVLink
  int x_by_row;
  // weight-gradient mode: K extent (token rows) and row base of each group
  const int32_t* k_rows;      // [G] or null -> k_rows_const
  int64_t k_rows_const;
  int64_t k_stride;
  float* Dacc;                // EPI_WGRAD_ACC output [P, N] fp32
  // dynamic tile scheduling: tiles are claimed in order with atomicAdd on this
  // (zeroed) counter by the leader's producer and handed to the pair's warps
  // through an smem queue, so the clusters that share a weight tile stay in step
  // (static round robin drifts and re-reads weights from HBM); null = static
  int* tile_counter;
  // A rows gathered by index: A row (g*row_stride + r) = X[a_gather[g*row_stride + r]]
  // through TMA tile::gather4 (map_a is then a {64, 1}-box map over X): the dispatch
  // copy of the k=1 layer is folded into GEMM1's producer
  const int32_t* a_gather;
  // Residual-MoE shared-MLP groups (see EPI_BIAS_RESID); zero-initialised = off
  int has_a2, a2_group;       // groups >= a2_group: A rows from map_a2, row (g-a2_group)*row_stride+r
  int has_rc, rc_group;       // groups >= rc_group: resid-combine epilogue, token rows as for A2
  const int32_t* c_ids;       // [S, k] routing of the combine
  const int32_t* c_slots;     // [S, k]
  const float* c_gp;          // [S, k]
  int c_k;
  int64_t c_cap;
  int64_t c_tokens;           // S
  int* c_done;                // zeroed: expert-tile epilogue warps done storing y
  const int32_t* c_row_index; // [S, k] row of y per choice (-1 dropped), or null: e*cap+slot
  // EP push return (EPI_BIAS / EPI_BIAS_COMBINE): valid row r is stored to rank
  // row_src[r]'s buffer push_base[row_src[r]] at row row_token[r] (over NVLink)
  void* const* push_base;
  const int32_t* row_src;
  // gate (CTA pairs): pair p owns the 128-row routing tiles [p*R/P, (p+1)*R/P), run
  // two per pair tile; an odd last one runs on the leader's rows only (the peer
  // skips its A load) - balanced to one routing tile instead of one pair tile
  int gate_bal;
  int coal_store;   // fused combine: stage each 32 x 32 chunk in smem, store 4 lanes per row
  int tma_store;    // EPI_BIAS / EPI_BIAS_GELU: whole-box TMA stores through map_d
  int stream_hint;  // epilogue outputs / residual reads are touched once: evict them first
  int raster;       // tile order (see tile_at)
  int prefetch;     // L2 prefetch of the next tile's streamed operand
  int prefetch_cur; // gate, single wave (decode sizes): L2 prefetch of the tile's K blocks past the ring
};

// CG = 1: one CTA computes a BM x BN tile (tcgen05.mma.cta_group::1, M=128).
// CG = 2: a 2-CTA cluster computes a (2*BM) x BN tile with cta_group::2 (M=256):
// each CTA loads its own 128 rows of A and BN/2 rows of B, the leader CTA issues
// the MMAs for the pair, each CTA's TMEM holds its 128 accumulator rows.
// Accumulator stages in TMEM (512 fp32 columns per lane): two (epilogue of
// tile i overlaps the MMAs of tile i+1) up to BN = 256; a BN = 512 tile (2-CTA
// 256 x 512, two N=256 MMAs per K step) fills TMEM, so it has one.
template <int BN>
constexpr int acc_stages() {
  return 2 * BN <= 512 ? 2 : 1;
}

// MS: 128-row A sub-tiles per CTA sharing each B stage (the gate: two pair tiles
// of tokens against one W_g^T stage, so the weight is streamed half as often)
template <int BN, int STAGES, int CG, int OUT = 0, int MS = 1>
struct Smem {
  static constexpr int kABytes = MS * BM * BK * 2;
  static constexpr int kBBytes = (BN / CG) * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOff = STAGES * kStageBytes;
  // full/empty ring, 2 x tfull/tempty, tmem slot, pbar ring, tile-queue full/empty
  // barriers and the tile-queue slots (dynamic scheduling)
  static constexpr int kBarBytes = (3 * STAGES + 8 + 2 * kTileQ) * 8 + 16 + kTileQ * 4;
  static constexpr int kTileOff = kBarOff + kBarBytes;
  static constexpr int kBiasOff = (kTileOff + (kMaxGroups + 1) * 4 + 127) / 128 * 128;  // AS x BN fp32
  // epilogue staging for TMA stores: OUT bytes, 1024-aligned
  static constexpr int kOutOff = (kBiasOff + acc_stages<BN>() * BN * 4 + 1023) / 1024 * 1024;
  static constexpr int kTotal = kOutOff + OUT + 1024;                    // +1024 align slack
};

template <int BN, int MS = 1>
constexpr uint32_t tmem_cols() {
  return (acc_stages<BN * MS>() * BN * MS) < 32 ? 32 : (acc_stages<BN * MS>() * BN * MS);
}

// EPI_WGRAD stages each warp's 32 x 32 output chunk in smem (2 x 2 KB per warp,
// 64-B swizzle: conflict-free row-per-lane writes) and TMA-stores it: the
// weight-gradient tiles have a short K (one expert's tokens), so the output
// stream is 4x denser per flop than the forward GEMMs and uncoalesced
// row-per-thread stores became the bottleneck.
// The forward expert GEMMs (EPI_BIAS / EPI_BIAS_GELU, 2-CTA) use the same
// staging when the caller marks the groups' padding rows as scratch
// (args.tma_store): bulk tensor stores instead of row-per-lane 16-B stores cut
// the L2 write transactions of the 1 GB GEMM1 output (energy: the kernel runs
// at the 1 kW cap).
// Staging buffers per epilogue warp: 2 (double-buffered) or 1 for BN = 512,
// whose 48 KB stages leave less room.
template <int BN>
constexpr int out_bufs() {
  return BN > 256 ? 1 : 2;
}
template <int EPI, int EW, int CG, int BN = 256>
constexpr int out_stage_bytes() {
  // (the 2-CTA fused-combine GEMM stages one 32 x 32 chunk per warp for the
  // coalesced row stores of the EP push return)
  return (EPI == EPI_WGRAD ||
          (CG == 2 && (EPI == EPI_BIAS || EPI == EPI_BIAS_GELU || EPI == EPI_BIAS_RESID)))
             ? EW * out_bufs<BN>() * 2048
             : ((CG == 2 && is_combine<EPI>()) ? EW * 2048 : 0);
}

// CL = cluster size: CG (one CTA pair per cluster) or 2*CG = 4: two pairs run the
// two m-blocks of the same (group, n-block) and share the weight tile, each CTA
// loading half of it and multicasting to its counterpart in the other pair.
// SUB: m-blocks a pair runs per scheduled tile (1, or 2 for the 2-CTA instance that
// shares a cluster-4 launch's tile pool, whose tiles span two m-blocks).
template <int BN, int STAGES, int EPI, int CG, int EW, int CL = CG, int SUB = 1, int MS = 1>
__global__ void __launch_bounds__(threads_for<EW, EPI>(), 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_d, GemmArgs args,
                        const __grid_constant__ CUtensorMap map_a2) {
  using L = Smem<BN, STAGES, CG, out_stage_bytes<EPI, EW, CG, BN>(), MS>;
  static_assert(MS == 1 || (EPI == EPI_GATE && CL == CG && SUB == 1), "A sub-tiles: gate pairs only");
  constexpr int TM = BM * CG;  // rows per MMA (a pair tile)
  constexpr int AS = acc_stages<BN * MS>();
  constexpr int kAccW = BN * MS;  // TMEM columns per accumulator stage
  // MMAs per K step: N <= 256 per tcgen05.mma; a BN = 512 pair tile issues two,
  // each CTA holding 128 B rows of each (two 16 KB halves of its B stage)
  constexpr int kNI = (CG == 2 && BN > 256) ? BN / 256 : 1;
  static_assert(kNI == 1 || (CG == 2 && BN == 512), "BN = 512 needs the 2-CTA pair");
  // BN = 512 forward tiles hand the accumulator over in kParts column parts of
  // kPW (tfull/tempty[j]; N = kPW MMAs) so the epilogue overlaps the MMAs
  // without a second accumulator buffer
  constexpr bool kSplit = kNI == 2 && (EPI == EPI_BIAS || EPI == EPI_BIAS_GELU || is_combine<EPI>());
  // (two N=256 halves: N=128 parts re-read A from smem twice as often and measured slower)
  constexpr int kParts = kSplit ? 2 : 1;
  constexpr int kPW = BN / kParts;
  constexpr bool kMN = EPI == EPI_WGRAD || EPI == EPI_WGRAD_ACC;  // MN-major operands
  extern __shared__ uint8_t smem_raw[];
  if (threadIdx.x == 0) GATE_TRACE(0);
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 4;  // [4]: accumulator stages, or the kSplit column parts
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  uint64_t* pbar = tempty + 5;  // [STAGES] weight-gradient partial K blocks (CTA-local)
  uint64_t* tq_full = pbar + STAGES;   // [kTileQ]
  uint64_t* tq_empty = tq_full + kTileQ;
  volatile int* tq = reinterpret_cast<volatile int*>(tq_empty + kTileQ);
  int32_t* tile_start = reinterpret_cast<int32_t*>(smem + L::kTileOff);

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int G = args.G;
  const int n_blocks = (args.N + BN - 1) / BN;
  static_assert(CL == CG || (CG == 2 && CL == 4), "cluster = one pair or two pairs");
  constexpr int CLP = CL / CG;  // CTA pairs per cluster
  constexpr int TMC = TM * CLP * SUB * MS;  // rows per scheduled tile
  const uint32_t qrank = CL > 1 ? cluster_ctarank() : 0;
  const uint32_t cta = qrank % CG;    // rank inside the CTA pair
  const uint32_t pair = qrank / CG;   // pair inside the cluster
  const uint32_t pl = qrank - cta;    // this pair's leader CTA
  const bool leader = cta == 0;
  const int work_id = blockIdx.x / CL, work_stride = gridDim.x / CL;
  if constexpr (CG == 2) cluster_sync();  // both CTAs resident before the paired TMEM alloc

  pdl_trigger();  // (programmatic dependent launch: see common.cuh)
  // ---- per-CTA tile table: tile_start[g] = sum_{g'<g} ceil(rows/TM) * n_blocks
  if (warp == 0) {
    pdl_wait();  // the group row counts come from the previous kernel
    const int per = (G + 31) / 32;
    const int g0 = lane * per;
    int local = 0;
    for (int g = g0; g < min(G, g0 + per); ++g) {
      const int64_t r = args.rows ? args.rows[g] : args.rows_const;
      local += (int)((r + TMC - 1) / TMC) * n_blocks;
    }
    int incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    int run = incl - local;
    for (int g = g0; g < min(G, g0 + per); ++g) {
      tile_start[g] = run;
      const int64_t r = args.rows ? args.rows[g] : args.rows_const;
      run += (int)((r + TMC - 1) / TMC) * n_blocks;
    }
    if (lane == 31) tile_start[G] = incl;
  }
  if (warp == 1) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], CG);  // CG=2: the peer's producer arrives remotely on the leader's
        mbar_init(&empty[s], CLP);  // CL=4: both pairs' MMAs release every stage
      }
      for (int a = 0; a < (kSplit ? kParts : AS); ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], EW * CG);  // every epilogue warp of the pair arrives
      }
      for (int s = 0; s < STAGES; ++s) mbar_init(&pbar[s], 1);
      // tile queue: full = the leader producer's (remote) arrive; empty (leader's) = every
      // consumer warp of the pair: MMA + epilogue (+ fix-up) warps, and the peer's producer
      constexpr int kFix = kMN ? 1 : 0;
      for (int q = 0; q < kTileQ; ++q) {
        mbar_init(&tq_full[q], 1);
        // the other CTAs' producers, the pairs' MMA warps, every epilogue / fix-up warp
        mbar_init(&tq_empty[q], (CL - 1) + CLP + (EW + kFix) * CL);
      }
      mbar_fence_init();
    }
    __syncwarp();
    if constexpr (CG == 2)
      tmem_alloc_cg2(tmem_slot, tmem_cols<BN, MS>());
    else
      tmem_alloc(tmem_slot, tmem_cols<BN, MS>());
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    if (args.has_a2) tma_prefetch(&map_a2);
    if (EPI == EPI_WGRAD || args.tma_store) tma_prefetch(&map_d);
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();  // barrier inits visible to the peer before any remote arrive
  else
    __syncthreads();
  tc_fence_after();
  pdl_wait();  // every role: no global access before the predecessor grid completed
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) GATE_TRACE(1);
  const int total_tiles = tile_start[G];

  // Work order: tiles are numbered (group, m block, n block) with n fastest and
  // each cluster takes runs of kRun consecutive tiles: kRun n-blocks of the same
  // activation rows, so the A tile its own SMs just streamed is re-read from L2
  // a tile later (temporal locality inside the cluster), while the clusters that
  // run the other m-blocks of the same n-blocks share each weight tile.
  // args.raster: 0 = plain round robin with m fastest (concurrent clusters share
  // the weight tile), 1 = round robin over runs of 4 n-blocks with n fastest.
  const int kRun = args.raster == 1 ? 4 : 1;
  auto tile_at = [&](int it) {
    return ((it / kRun) * work_stride + work_id) * kRun + (it % kRun);
  };
  // tile -> (group, m block, n block)
  auto decode = [&](int tile, int& g, int& mb, int& nb) {
    while (tile_start[g + 1] <= tile) ++g;
    const int local = tile - tile_start[g];
    const int64_t r = args.rows ? args.rows[g] : args.rows_const;
    if (args.raster == 1) {
      mb = local / n_blocks;
      nb = local - mb * n_blocks;
    } else {
      const int mblocks = (int)((r + TMC - 1) / TMC);
      nb = local / mblocks;
      mb = local - nb * mblocks;
    }
  };

  // next tile for loop iteration `it` (whole warp), -1 when done. Static: round
  // robin. Dynamic: the leader's producer claims tiles and publishes them to both
  // CTAs' queues; every other role reads its CTA's queue and frees the slot.
  const bool dyn = args.tile_counter != nullptr;
  int claimed = -1;  // writer (lane 0): the tile claimed one iteration ahead
  // balanced gate: "tiles" are first routing tiles (128-row units) of this pair's range
  const bool gbal = EPI == EPI_GATE && CL == CG && args.gate_bal != 0;
  int g_lo = 0, g_hi = 0;
  if (gbal) {
    const int R = (int)((args.S + BM - 1) / BM);
    g_lo = (int)((int64_t)work_id * R / work_stride);
    g_hi = (int)((int64_t)(work_id + 1) * R / work_stride);
  }
  auto fetch = [&](int it, bool writer) -> int {
    if (gbal) {
      const int t = g_lo + 2 * it;
      return t < g_hi ? t : -1;
    }
    if (!dyn) {
      const int t = tile_at(it);
      return t < total_tiles ? t : -1;
    }
    const int slot = it % kTileQ;
    const uint32_t ph = (uint32_t)(it / kTileQ) & 1u;
    int t = 0;
    if (writer) {
      mbar_wait(&tq_empty[slot], ph ^ 1u);
      if (lane == 0) {
        // claim one tile ahead: the atomic's round trip overlaps this tile's loads
        if (it == 0) claimed = atomicAdd(args.tile_counter, 1);
        t = claimed < total_tiles ? claimed : -1;
        if (t >= 0) claimed = atomicAdd(args.tile_counter, 1);
        tq[slot] = t;
#pragma unroll
        for (int r = 1; r < CL; ++r) {  // every other CTA of the cluster
          st_shared_cluster_i32(const_cast<int*>(&tq[slot]), r, t);
          mbar_arrive_cluster_release(&tq_full[slot], r);
        }
        mbar_arrive(&tq_full[slot]);
      }
      t = __shfl_sync(0xffffffffu, t, 0);
    } else {
      mbar_wait(&tq_full[slot], ph);
      t = tq[slot];
      __syncwarp();
      if (lane == 0) {
        if (qrank != 0)
          mbar_arrive_cluster_release(&tq_empty[slot], 0);
        else
          mbar_arrive(&tq_empty[slot]);
      }
    }
    return t;
  };

  if (warp == 0) {
    // ===================== TMA producer (both CTAs of a pair load their halves)
    int stage = 0;
    uint32_t phase = 0;
    int g = 0;
    const int num_kb = (args.K + BK - 1) / BK;
    // (L2 eviction-priority hints on A/B were measured and removed: evict_first
    // on the weights raised DRAM traffic from 6.2 to 9.1 GB per GEMM1 launch)
    int gp = 0;  // group cursor for the prefetch look-ahead
    int cur = -1;
    for (int vit = 0;; ++vit) {
      const int sub = vit % SUB;
      if (sub == 0) cur = fetch(vit / SUB, qrank == 0);
      const int tile = cur;
      const int it = vit / SUB;
      if (tile < 0) break;
      int mb = 0, nb = 0;
      if (!gbal) decode(tile, g, mb, nb);
      const int64_t rs = args.row_start ? args.row_start[g] : (int64_t)g * args.row_stride;
      const int w = args.weight_idx ? args.weight_idx[g] : g;
      const int mrow = gbal ? tile * BM : mb * TMC + (int)(pair * SUB + sub) * TM;  // this pair's m-block
      // (the per-tile TMA coordinates are made warp-uniform with a lane-0 shuffle, so
      // ptxas keeps the issue path on uniform registers: no per-load R2UR waterfall)
      // balanced gate, odd last routing tile: only the leader's 128 rows are this pair's
      const bool g_half = __shfl_sync(0xffffffffu, (int)(gbal && tile + 1 >= g_hi), 0) != 0;
      // shared-MLP groups of a Residual-MoE launch read x (map_a2) instead of the
      // dispatched expert buffer
      const bool use_a2 = __shfl_sync(0xffffffffu, (int)(args.has_a2 && g >= args.a2_group), 0) != 0;
      const CUtensorMap* mA = use_a2 ? &map_a2 : &map_a;
      const int64_t rs_a = use_a2 ? (int64_t)(g - args.a2_group) * args.row_stride : rs;
      const int a_row = __shfl_sync(0xffffffffu, (int)(rs_a + (int64_t)mrow + cta * BM), 0);
      const int b_base = __shfl_sync(0xffffffffu, w * args.N + nb * BN, 0);
      const int b_row = b_base + cta * (BN / CG);
      // gather mode: this lane's 4 source rows of the CTA's 128-row A tile (rows past
      // the group's count read row 0: their outputs are padding)
      int grow[4] = {0, 0, 0, 0};
      if (!kMN && args.a_gather != nullptr) {
        const int64_t rg = args.rows ? args.rows[g] : args.rows_const;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t lr = (int64_t)mrow + cta * BM + 4 * lane + i;
          grow[i] = lr < rg ? args.a_gather[rs + lr] : 0;
        }
      }
      if (args.prefetch && !dyn && gbal && lane == 0) {
        // balanced gate: the next routing-tile pair of this pair's range (an odd last
        // routing tile is the leader's alone)
        const int nt = tile + 2;
        if (nt < g_hi && (cta == 0 || nt + 1 < g_hi)) {
          const int pa = (nt + (int)cta) * BM;
          for (int kb = 0; kb < num_kb; ++kb) tma_prefetch_l2_2d(&map_a, kb * BK, pa);
        }
      }
      if (args.prefetch && !dyn && !gbal && lane == 0) {
        // Warm L2 with the NEXT tile's streamed operand while this one runs: the
        // smem ring alone keeps too few DRAM bytes in flight per SM to hide the
        // loaded HBM latency (x for the gate, the weights for the expert GEMMs).
        const int nt = tile_at(it + 1);
        if (nt < total_tiles) {
          int pm, pn;
          if (gp < g) gp = g;
          decode(nt, gp, pm, pn);
          if (EPI == EPI_GATE) {
            const int64_t prs = args.row_start ? args.row_start[gp] : (int64_t)gp * args.row_stride;
            const int pa = (int)(prs + (int64_t)pm * TM + cta * BM);
            for (int kb = 0; kb < num_kb; ++kb) tma_prefetch_l2_2d(&map_a, kb * BK, pa);
          } else {
            const int pw = args.weight_idx ? args.weight_idx[gp] : gp;
            const int pb = pw * args.N + pn * BN + cta * (BN / CG);
            for (int kb = 0; kb < num_kb; ++kb) tma_prefetch_l2_2d(&map_b, kb * BK, pb);
          }
        }
      }
      int kb_end = num_kb;
      int kg = 0;
      if constexpr (kMN) {
        kg = (int)(args.k_rows ? args.k_rows[g] : args.k_rows_const);
        kb_end = (kg + BK - 1) / BK;
      }
      for (int kb = 0; kb < kb_end; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0 && vit == 0 && kb == 0) GATE_TRACE(2);
        if constexpr (kMN) {
          // X^T / Y^T tiles: boxes of 64 MN columns x 64 token rows (one 128-B
          // line per row); A = this CTA's BM columns of X, B = its BN/CG of Y
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          const int krow = (int)((int64_t)g * args.k_stride + (int64_t)kb * BK);
          const int pa = mb * TM + cta * BM;
          const int pb = nb * BN + cta * (BN / CG);
          constexpr int kBoxB = (BN / CG) / 64;
          const int rem = kg - kb * BK;
          if (rem >= BK) {
            if (lane == 0) {
              if constexpr (CG == 2) {
#pragma unroll
                for (int j = 0; j < 2; ++j) tma_load_2d_cg2(sa + j * 8192, &map_a, &full[stage], pa + 64 * j, krow);
#pragma unroll
                for (int j = 0; j < kBoxB; ++j) tma_load_2d_cg2(sb + j * 8192, &map_b, &full[stage], pb + 64 * j, krow);
                if (leader)
                  mbar_arrive_expect_tx(&full[stage], CG * L::kStageBytes);
                else
                  mbar_arrive_cluster(&full[stage], pl);
              } else {
                mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
#pragma unroll
                for (int j = 0; j < 2; ++j) tma_load_2d(sa + j * 8192, &map_a, &full[stage], pa + 64 * j, krow);
#pragma unroll
                for (int j = 0; j < kBoxB; ++j) tma_load_2d(sb + j * 8192, &map_b, &full[stage], pb + 64 * j, krow);
              }
            }
          } else {
            // last, partial K block: rows >= rem belong to padding (or the next
            // group) and may hold anything, NaN included. Load into this CTA's smem
            // on the stage's local barrier; the fix-up warp zeroes those rows and
            // then releases the stage to the MMA (the producer does not stall)
            if (lane == 0) {
              mbar_arrive_expect_tx(&pbar[stage], L::kStageBytes);
#pragma unroll
              for (int j = 0; j < 2; ++j) tma_load_2d(sa + j * 8192, &map_a, &pbar[stage], pa + 64 * j, krow);
#pragma unroll
              for (int j = 0; j < kBoxB; ++j) tma_load_2d(sb + j * 8192, &map_b, &pbar[stage], pb + 64 * j, krow);
            }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          continue;
        }
        if (args.a_gather != nullptr) {
          // A: 32 lanes x gather4 (4 rows x 128 B each); B: one tile load
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          if constexpr (CG == 2) {
            tma_gather4_cg2(sa + 512 * lane, &map_a, &full[stage], kb * BK, grow[0], grow[1],
                            grow[2], grow[3]);
            if (lane == 0) {
              if constexpr (kNI > 1) {
#pragma unroll
                for (int i = 0; i < kNI; ++i)
                  tma_load_2d_cg2(sb + i * 128 * BK * 2, &map_b, &full[stage], kb * BK,
                                  w * args.N + nb * BN + i * 256 + (int)cta * 128);
              } else {
                tma_load_2d_cg2(sb, &map_b, &full[stage], kb * BK, b_row);
              }
              if (leader)
                mbar_arrive_expect_tx(&full[stage], CG * L::kStageBytes);
              else
                mbar_arrive_cluster(&full[stage], pl);
            }
          } else {
            if (lane == 0) mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
            __syncwarp();
            tma_gather4(sa + 512 * lane, &map_a, &full[stage], kb * BK, grow[0], grow[1], grow[2],
                        grow[3]);
            if (lane == 0) tma_load_2d(sb, &map_b, &full[stage], kb * BK, b_row);
          }
        } else {  // warp-uniform: every lane runs this, one elected lane issues (*_e)
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          if constexpr (kNI > 1 && CL == 4) {
            // 256 x 512 pair tiles, two pairs per cluster on the two m-blocks of one
            // (group, n-block): the 512-column weight tile is shared - every CTA loads
            // half of its B rows of each MMA and multicasts them to its counterpart
            // in the other pair (L2->SM weight bytes halved again)
            tma_load_2d_cg2_e(sa, mA, &full[stage], kb * BK, a_row);
            constexpr int kHalf = 128 / CLP;  // B rows per multicast box
#pragma unroll
            for (int i = 0; i < kNI; ++i)
              tma_load_2d_cg2_mc_e(sb + i * 128 * BK * 2 + pair * kHalf * BK * 2, &map_b,
                                 &full[stage], kb * BK,
                                 b_base + i * 256 + (int)cta * 128 + (int)pair * kHalf,
                                 (uint16_t)((1u << cta) | (1u << (cta + 2))));
            if (leader)
              mbar_arrive_expect_tx_e(&full[stage], CG * L::kStageBytes);
            else
              mbar_arrive_cluster_e(&full[stage], pl);
          } else if constexpr (kNI > 1) {
            tma_load_2d_cg2_e(sa, mA, &full[stage], kb * BK, a_row);
#pragma unroll
            for (int i = 0; i < kNI; ++i)  // B rows of MMA i: [nb*BN + i*256 + cta*128, +128)
              tma_load_2d_cg2_e(sb + i * 128 * BK * 2, &map_b, &full[stage], kb * BK,
                              b_base + i * 256 + (int)cta * 128);
            if (leader)
              mbar_arrive_expect_tx_e(&full[stage], CG * L::kStageBytes);
            else
              mbar_arrive_cluster_e(&full[stage], pl);
          } else if constexpr (CL == 4) {
            // weight tile shared by both pairs: load my half of my 128 B rows and
            // multicast it to my counterpart in the other pair (same cta index)
            tma_load_2d_cg2_e(sa, mA, &full[stage], kb * BK, a_row);
            constexpr int kHalf = BN / CG / CLP;  // B rows per multicast box
            tma_load_2d_cg2_mc_e(sb + pair * kHalf * BK * 2, &map_b, &full[stage], kb * BK,
                               b_row + pair * kHalf, (uint16_t)((1u << cta) | (1u << (cta + 2))));
            if (leader)
              mbar_arrive_expect_tx_e(&full[stage], CG * L::kStageBytes);
            else
              mbar_arrive_cluster_e(&full[stage], pl);
          } else if constexpr (CG == 2) {
            // (balanced gate half tile: the peer's A rows belong to the next pair - not
            // loaded; the MMA's rows for them are garbage the epilogue ignores)
            if (!(g_half && cta == 1)) {
#pragma unroll
              for (int ms = 0; ms < MS; ++ms)  // sub-tile ms: the pair tile ms*TM rows on
                tma_load_2d_cg2_e(sa + ms * BM * BK * 2, mA, &full[stage], kb * BK, a_row + ms * TM);
            }
            tma_load_2d_cg2_e(sb, &map_b, &full[stage], kb * BK, b_row);
            if (leader)
              mbar_arrive_expect_tx_e(&full[stage], CG * L::kStageBytes - (g_half ? L::kABytes : 0));
            else
              mbar_arrive_cluster_e(&full[stage], pl);
          } else {
            mbar_arrive_expect_tx_e(&full[stage], L::kStageBytes);
            tma_load_2d_e(sa, mA, &full[stage], kb * BK, a_row);
            tma_load_2d_e(sb, &map_b, &full[stage], kb * BK, b_row);
          }
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only). The whole warp runs the
    // loop with warp-uniform values and one elected lane issues each tcgen05 op
    // (the *_e helpers), so descriptors stay in uniform registers
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
    constexpr uint32_t idesc = kMN ? make_idesc_bf16_mn(TM, BN) : make_idesc_bf16(TM, BN / kNI);
    // K step of one MMA (16 elements): +32 B inside the swizzle line (K-major) or
    // two 8-row groups (+2048 B, MN-major); descriptor units are 16 B
    constexpr uint64_t kStep = kMN ? 128 : 2;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int num_kb = (args.K + BK - 1) / BK;
    int g = 0;
    int cur = -1;
    for (int vit = 0; leader; ++vit) {
      if (vit % SUB == 0) cur = fetch(vit / SUB, false);
      const int tile = __shfl_sync(0xffffffffu, cur, 0);
      if (tile < 0) break;
      int kb_end = num_kb;
      if constexpr (kMN) {
        int mb_, nb_;
        decode(tile, g, mb_, nb_);
        const int64_t kg = args.k_rows ? args.k_rows[g] : args.k_rows_const;
        kb_end = (int)((kg + BK - 1) / BK);  // 0 for an empty group: the epilogue writes zeros
        kb_end = __shfl_sync(0xffffffffu, kb_end, 0);
      }
      if constexpr (kSplit) {
        // BN = 512 pair tile, TMEM full: the accumulator is handed over in kParts
        // column parts (MMAs of N = kPW, each CTA holding kPW/2 B rows of a part).
        // First kRA K blocks: parts 0.. run ahead while the epilogue still drains the
        // later parts of the previous tile; last kRA K blocks: part by part, so the
        // epilogue of part j overlaps the tail MMAs of parts j+1...
        constexpr uint32_t idesc_p = make_idesc_bf16(TM, kPW);
        const int s0 = stage;
        const uint32_t ph0 = phase;
        auto wait_kb = [&](int kb) {
          mbar_wait(&full[(s0 + kb) % STAGES], ph0 ^ (uint32_t)(((s0 + kb) / STAGES) & 1));
          tc_fence_after();
        };
        auto mma_part = [&](int kb, int j) {
          const uint8_t* sa = smem + ((s0 + kb) % STAGES) * L::kStageBytes;
          const uint64_t adesc = make_sdesc_sw128(sa);
          const uint64_t bdesc =
              make_sdesc_sw128(sa + L::kABytes) + (uint64_t)j * (((kPW / 2) * BK * 2) >> 4);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16_cg2_e(tmem_u + j * kPW, adesc + kStep * kk, bdesc + kStep * kk, idesc_p,
                            (kb | kk) != 0);
        };
        auto release = [&](int kb) {
          umma_commit_cg2_e(&empty[(s0 + kb) % STAGES], CL == 4 ? 0xF : 0x3);
        };
        constexpr int kRA = STAGES - 1;
        const int ra = kb_end < kRA ? kb_end : kRA;
        const int c0 = kb_end - kRA > ra ? kb_end - kRA : ra;
        for (int j = 0; j < kParts; ++j) {
          mbar_wait(&tempty[j], acc_phase ^ 1);
          tc_fence_after();
          for (int kb = 0; kb < ra; ++kb) {
            if (j == 0) wait_kb(kb);
            mma_part(kb, j);
            if (j == kParts - 1) release(kb);
          }
        }
        for (int kb = ra; kb < c0; ++kb) {
          wait_kb(kb);
#pragma unroll
          for (int j = 0; j < kParts; ++j) mma_part(kb, j);
          release(kb);
        }
        for (int j = 0; j < kParts; ++j) {
          for (int kb = c0; kb < kb_end; ++kb) {
            if (j == 0) wait_kb(kb);
            mma_part(kb, j);
            if (j == kParts - 1) release(kb);
          }
          umma_commit_cg2_e(&tfull[j], (uint16_t)(0x3u << pl));
        }
        __syncwarp();
        stage = (s0 + kb_end) % STAGES;
        phase = ph0 ^ (uint32_t)(((s0 + kb_end) / STAGES) & 1);
        acc_phase ^= 1;
        continue;
      }
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_u + acc * kAccW;
      for (int kb = 0; kb < kb_end; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0 && vit == 0 && kb == 0) GATE_TRACE(3);
        if (lane == 0 && vit == 0 && kb == kb_end - 1) GATE_TRACE(4);
        const uint8_t* sa = smem + stage * L::kStageBytes;
        const uint8_t* sb = sa + L::kABytes;
        const uint64_t adesc = kMN ? make_sdesc_sw128_mn(sa) : make_sdesc_sw128(sa);
        const uint64_t bdesc = kMN ? make_sdesc_sw128_mn(sb) : make_sdesc_sw128(sb);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          if constexpr (kNI > 1) {
#pragma unroll
            for (int i = 0; i < kNI; ++i)  // B half i = 128 rows x 128 B further (>>4: +1024)
              umma_bf16_cg2_e(d_tmem + i * 256, adesc + kStep * kk,
                              bdesc + (uint64_t)i * ((128 * BK * 2) >> 4) + kStep * kk, idesc,
                              (kb | kk) != 0);
          } else if constexpr (CG == 2) {
#pragma unroll
            for (int ms = 0; ms < MS; ++ms)
              umma_bf16_cg2_e(d_tmem + ms * BN,
                              adesc + (uint64_t)ms * ((BM * BK * 2) >> 4) + kStep * kk,
                              bdesc + kStep * kk, idesc, (kb | kk) != 0);
          } else {
            umma_bf16_e(d_tmem, adesc + kStep * kk, bdesc + kStep * kk, idesc, (kb | kk) != 0);
          }
        }
        if constexpr (CG == 2)
          umma_commit_cg2_e(&empty[stage], CL == 4 ? 0xF : 0x3);  // frees the stage (all CTAs that wrote it)
        else
          umma_commit_e(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if constexpr (CG == 2)
        umma_commit_cg2_e(&tfull[acc], (uint16_t)(0x3u << pl));
      else
        umma_commit_e(&tfull[acc]);
      if (++acc == AS) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp < 2 + EW) {
    // ===================== epilogue warps 2..2+EW-1
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    constexpr int kColSplit = EW / 4;    // warps sharing a quarter split the columns
    const int col_part = (int)(warp - 2) / 4;          // 0 .. kColSplit-1
    constexpr int kChunks = BN / 32 / kColSplit;       // 32-column chunks per warp
    const int row_in_tile = pair * TM + cta * BM + quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    int g = 0;
    const int N = args.N;
    const uint64_t pol_stream = policy_evict_first();
    int ostage = 0;  // EPI_WGRAD staging buffer toggle
    (void)ostage;
    if constexpr (EPI == EPI_GATE) {
      if (args.probsum != nullptr) {
        float* psum = reinterpret_cast<float*>(smem + L::kTileOff) + 8 + 4 * args.E;
        for (int i = (warp - 2) * 32 + lane; i < args.E; i += 128) psum[i] = 0.f;
        named_bar_sync(1, 128);
      }
    }
    int cur = -1;
    for (int vit = 0;; ++vit) {
      const int sub = vit % SUB;
      if (sub == 0) cur = fetch(vit / SUB, false);
      const int tile = cur;
      if (tile < 0) break;
      int mb = 0, nb = 0;
      if (!gbal) decode(tile, g, mb, nb);
      const int64_t rs = args.row_start ? args.row_start[g] : (int64_t)g * args.row_stride;
      const int64_t rows_g = args.rows ? args.rows[g] : args.rows_const;
      const int w = args.weight_idx ? args.weight_idx[g] : g;
      const int64_t local_row =
          gbal ? (int64_t)tile * BM + row_in_tile : (int64_t)mb * TMC + sub * TM + row_in_tile;
      const bool g_skip = gbal && cta == 1 && tile + 1 >= g_hi;  // the next pair's rows
      const bool valid = local_row < rows_g && !g_skip;
      const int64_t out_row = rs + local_row;
      bool kzero = false;  // weight gradient of a group with no rows: zeros, TMEM not written
      if constexpr (kMN) kzero = (args.k_rows ? args.k_rows[g] : args.k_rows_const) == 0;
      if constexpr (EPI == EPI_GATE) {
        if (args.prefetch_cur && warp == 2 && lane == 0) {
          // one tile per CTA (decode-sized batches): while the producer issues the
          // ring's first loads, this (still idle) warp requests the K blocks the ring
          // cannot hold yet into L2, so the ring refills from L2 instead of paying a
          // DRAM round trip per stage (this CTA's x rows and its W_g^T rows)
          const int a_row = (int)(rs + (int64_t)mb * TMC + sub * TM + pair * TM + cta * BM);
          const int b_row = w * args.N + nb * BN + cta * (BN / CG);
          const int num_kb = (args.K + BK - 1) / BK;
          for (int kb = STAGES; kb < num_kb; ++kb) {
            tma_prefetch_l2_2d(&map_a, kb * BK, a_row);
            tma_prefetch_l2_2d(&map_b, kb * BK, b_row);
          }
        }
      }

      mbar_wait(&tfull[kSplit ? 0 : acc], acc_phase);
      if (warp == 2 && lane == 0 && vit == 0) GATE_TRACE(5);
      tc_fence_after();
      // TMEM column and tile column of this warp's 32-column chunk c. kSplit: chunks
      // 2j, 2j+1 lie in column part j (handed over separately); part j's first
      // kPW/2 columns come from the leader's B rows, the rest from the peer's
      // (B rows of half h = j/2 map to tile columns h*256 + cta*128 + ...)
      constexpr int kCP = kChunks / kParts;  // chunks per part per warp
      auto tmem_col = [&](int c) -> int {
        return kSplit ? (c / kCP) * kPW + col_part * (kPW / 2) + (c % kCP) * 32
                      : (col_part * kChunks + c) * 32;
      };
      auto chunk_col = [&](int c) -> int {
        const int rr = (c / kCP) * (kPW / 2) + (c % kCP) * 32;  // B row in CTA col_part
        return kSplit ? (rr / 128) * 256 + col_part * 128 + rr % 128 : (col_part * kChunks + c) * 32;
      };
      const uint32_t t_lane = tmem_base + ((quarter * 32) << 16) + acc * kAccW;
      const uint32_t t_addr0 = tmem_base + ((quarter * 32) << 16) + acc * kAccW +
                              (EPI != EPI_GATE ? col_part * kChunks * 32 : 0);

      if constexpr (EPI != EPI_GATE) {
        const bool vec_ok = (N % 8) == 0;
        // the tile's BN bias values, staged once in smem by the epilogue warps
        // (double-buffered by accumulator index, so one barrier per tile)
        float* sbias = reinterpret_cast<float*>(smem + L::kBiasOff) + acc * BN;
        {
          const float* bias = args.bias ? args.bias + (int64_t)w * N : nullptr;
          for (int i = (warp - 2) * 32 + lane; i < BN; i += EW * 32) {
            const int col = nb * BN + i;
            // EPI_BIAS_GELU stages b/2: its epilogue works on w = (acc + b)/2 (exact)
            sbias[i] = (bias != nullptr && col < N) ? __ldg(bias + col) * (EPI == EPI_BIAS_GELU ? 0.5f : 1.f)
                                                    : 0.f;
          }
          named_bar_sync(2, EW * 32);
        }
        __nv_bfloat16* drow = args.D + out_row * N;
        // (push launches use <= 256-column tiles: no push code in the 512-column ones)
        const bool push = BN <= 256 && (EPI == EPI_BIAS || EPI == EPI_COMBINE_PUSH) &&
                          args.push_base != nullptr && valid;
        if (push && EPI == EPI_BIAS)
          drow = static_cast<__nv_bfloat16*>(args.push_base[args.row_src[out_row]]) +
                 (int64_t)args.row_token[out_row] * N;
        const __nv_bfloat16* xrow = nullptr;
        float prob = 0.f;
        __nv_bfloat16* arow = nullptr;  // EPI_GELU_SAVE: pre-activation output row
        if constexpr (is_combine<EPI>()) {
          const int64_t tok = valid ? args.row_token[out_row] : 0;
          prob = valid ? args.row_prob[out_row] : 0.f;
          drow = args.out + (args.x_by_row ? out_row : tok) * N;
          xrow = args.x_resid + (args.x_by_row ? out_row : tok) * N;
          if (push)  // the combined row goes straight to its source's output (NVLink)
            drow = static_cast<__nv_bfloat16*>(args.push_base[args.row_src[out_row]]) + tok * N;
        }
        if constexpr (EPI == EPI_GELU_BWD) xrow = args.x_resid + out_row * N;
        if constexpr (EPI == EPI_GELU_SAVE) arow = args.out + out_row * N;
        // EPI_BIAS_RESID, shared-MLP group: this row is token c_t; its kept expert rows
        // (ascending expert id, forward_layer's order, arch.py:399-410) and probabilities
        const bool rc = EPI == EPI_BIAS_RESID && args.has_rc && g >= args.rc_group;
        int64_t c_t = 0, cr0 = 0, cr1 = 0;
        float cp0 = 0.f, cp1 = 0.f;
        int cn = 0;
        if constexpr (EPI == EPI_BIAS_RESID) {
          if (rc) {
            // every expert tile's y must be stored first: the expert tiles precede the
            // shared ones in tile order and every CTA runs its tiles in order, so they
            // are all claimed by running CTAs and complete without waiting on this one
            const int expected = tile_start[args.rc_group] * EW * CG;
            if (lane == 0) {
              while (ld_acquire_gpu(args.c_done) < expected) __nanosleep(256);
            }
            __syncwarp();
            c_t = (int64_t)(g - args.rc_group) * args.row_stride + local_row;
            if (valid) {
              int e0 = 0;
              for (int j = 0; j < args.c_k; ++j) {
                int64_t r;
                if (args.c_row_index != nullptr) {
                  r = args.c_row_index[c_t * args.c_k + j];
                  if (r < 0) continue;
                } else {
                  const int sl = args.c_slots[c_t * args.c_k + j];
                  if (sl < 0) continue;
                  r = (int64_t)args.c_ids[c_t * args.c_k + j] * args.c_cap + sl;
                }
                const int e = args.c_ids[c_t * args.c_k + j];
                const float pj = args.c_gp[c_t * args.c_k + j];
                if (cn == 0) { cr0 = r; cp0 = pj; e0 = e; }
                else if (e < e0) { cr1 = cr0; cp1 = cp0; cr0 = r; cp0 = pj; }
                else { cr1 = r; cp1 = pj; }
                ++cn;
              }
            }
            drow = args.out + c_t * N;
            xrow = args.x_resid + c_t * N;
          }
        }
        constexpr bool kLoadX = is_combine<EPI>() || EPI == EPI_GELU_BWD;
        // residual row chunks (COMBINE) are prefetched one chunk ahead
        auto load_x = [&](int c, uint4 (&xq)[4]) {
          const int col0 = nb * BN + chunk_col(c);
          if (valid && vec_ok && col0 + 32 <= N) {
            const uint4* xs = reinterpret_cast<const uint4*>(xrow + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              xq[q] = args.stream_hint ? ld_global_nc_hint(xs + q, pol_stream) : __ldg(xs + q);
          }
        };
        // kStream (the fused combine on 256 x 512 tiles): not MUFU-bound, so chunks
        // are read one at a time and each part is handed back after its last chunk
        // (32 accumulator registers instead of a whole part: no spills)
        constexpr bool kStream = kSplit && is_combine<EPI>();
        // kStream: a part's residual chunks are all
        // loaded before the part's accumulator is awaited (the loads hide under the
        // MMAs; per-chunk prefetch left ~3 us of latency per part exposed, stalling
        // the MMA run-ahead); otherwise prefetched one chunk ahead
        constexpr int kXB = kStream ? kCP : 2;
        uint4 xbuf[kXB][4];
        auto xslot = [&](int c) -> int { return kStream ? c % kCP : c & 1; };
        if constexpr (kLoadX) {
          if constexpr (kStream) {
#pragma unroll
            for (int e = 0; e < kCP; ++e) load_x(e, xbuf[e]);
          } else {
            load_x(0, xbuf[0]);
          }
        }
        // TMEM loads double-buffered across 32-column chunks: the load of
        // chunk c+1 is in flight while chunk c is biased, activated and stored.
        // kSplit: a whole part is read into registers (kCP x 32 columns) and its
        // TMEM handed straight back, so the MMAs refill it while the epilogue
        // computes (the GELU drain is MUFU-bound and outlasts the MMA run-ahead)
        constexpr int kRB = kSplit ? (kStream ? 1 : kCP) : 2;
        uint32_t r[kRB][32];
        if constexpr (!kSplit) tmem_ld_32x32b_x32(t_lane + tmem_col(0), r[0]);
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          const int cl = chunk_col(c);  // column inside the tile
          const int col0 = nb * BN + cl;
          if constexpr (kLoadX && !kStream) {
            if (c + 1 < kChunks) load_x(c + 1, xbuf[(c + 1) & 1]);
          }
          if constexpr (kStream) {
            if (c % kCP == 0 && c > 0) {
              if constexpr (kLoadX) {
#pragma unroll
                for (int e = 0; e < kCP; ++e) load_x(c + e, xbuf[e]);
              }
              mbar_wait(&tfull[c / kCP], acc_phase);
              tc_fence_after();
            }
            tmem_ld_32x32b_x32(t_lane + tmem_col(c), r[0]);
            tmem_ld_wait_regs(r[0]);
            if (c % kCP == kCP - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(&tempty[c / kCP], pl);
            }
          } else if constexpr (kSplit) {
            if (c % kCP == 0) {
              if (c > 0) {
                mbar_wait(&tfull[c / kCP], acc_phase);
                tc_fence_after();
              }
#pragma unroll
              for (int e = 0; e < kCP; ++e) tmem_ld_32x32b_x32(t_lane + tmem_col(c + e), r[e]);
#pragma unroll
              for (int e = 0; e < kCP; ++e) tmem_ld_wait_regs(r[e]);
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(&tempty[c / kCP], pl);
            }
          } else {
            tmem_ld_wait_regs(r[c & 1]);
            if (c + 1 < kChunks) tmem_ld_32x32b_x32(t_lane + tmem_col(c + 1), r[(c + 1) & 1]);
          }
          // whole warp: 32 rows x 32 columns -> smem (row = lane, 64 B, 64-B swizzle)
          // -> one TMA tensor store; rows / columns past the group's block are
          // clipped by the 3-D map (N, rows per group, G)
          auto stage_store = [&](const uint32_t (&pk32)[16]) {
            constexpr int OB = out_bufs<BN>();
            uint8_t* ob = smem + L::kOutOff + ((warp - 2) * OB + (ostage % OB)) * 2048;
            if (lane == 0) bulk_wait_group_read<OB - 1>();  // this buffer's last store has read it
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int chunk = q ^ ((lane >> 1) & 3);  // SWIZZLE_64B
              *reinterpret_cast<uint4*>(ob + lane * 64 + chunk * 16) =
                  make_uint4(pk32[4 * q], pk32[4 * q + 1], pk32[4 * q + 2], pk32[4 * q + 3]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_3d(&map_d, ob, col0, (int)(mb * TMC + sub * TM + row_in_tile - lane), g);
              bulk_commit_group();
            }
            ++ostage;
          };
          if constexpr (EPI == EPI_WGRAD) {
            if (col0 < N) {
              uint32_t pk32[16];
#pragma unroll
              for (int i = 0; i < 16; ++i)
                pk32[i] = kzero ? 0u
                                : pack_bf16x2(__uint_as_float(r[c % kRB][2 * i]),
                                              __uint_as_float(r[c % kRB][2 * i + 1]));
              stage_store(pk32);
            }
            continue;
          }
          constexpr bool kTmaEpi = out_stage_bytes<EPI, EW, CG, BN>() > 0 && EPI != EPI_WGRAD &&
                                   !is_combine<EPI>();
          // EP push return: rows go to scattered peer rows, so the warp stages its
          // 32 x 32 chunk in smem and stores it 4 lanes per row (full 64-B row
          // segments per NVLink write instead of 16-B pieces of 32 different rows)
          // (also the local fused combine, whose rows are scattered over `out` by token:
          // 4x fewer store transactions, and the 256 x 512 tile's epilogue fits the
          // MMA run-ahead)
          constexpr bool kCoalOK = out_stage_bytes<EPI, EW, CG, BN>() > 0 &&
                                   ((EPI == EPI_BIAS && BN <= 256) || is_combine<EPI>());
          const bool coal = kCoalOK && (args.push_base != nullptr || (is_combine<EPI>() && args.coal_store)) &&
                            vec_ok && col0 + 32 <= N;
          if (col0 >= N) continue;
          if (!valid && !(kTmaEpi && args.tma_store) && !coal) continue;
          float v[32];
          const float4* b4 = reinterpret_cast<const float4*>(sbias + cl);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 bq = b4[q];
            constexpr float sc = EPI == EPI_BIAS_GELU ? 0.5f : 1.f;
            v[4 * q + 0] = fmaf(__uint_as_float(r[c % kRB][4 * q + 0]), sc, bq.x);
            v[4 * q + 1] = fmaf(__uint_as_float(r[c % kRB][4 * q + 1]), sc, bq.y);
            v[4 * q + 2] = fmaf(__uint_as_float(r[c % kRB][4 * q + 2]), sc, bq.z);
            v[4 * q + 3] = fmaf(__uint_as_float(r[c % kRB][4 * q + 3]), sc, bq.w);
          }
          if constexpr (EPI == EPI_BIAS_RESID) {
            if (rc) {  // out[t] = (x[t] + sum_j p_j y_j) + (acc + b2), arch.py:389-391
              if (!valid) continue;
              const __nv_bfloat16* y0r = args.D + cr0 * N;
              const __nv_bfloat16* y1r = args.D + cr1 * N;
              if (vec_ok && col0 + 32 <= N) {
                uint4 xq[4], aq[4], bq[4];
                const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  xq[q] = __ldg(reinterpret_cast<const uint4*>(xrow + col0) + q);
                  // y was stored by this launch's expert tiles: L2-coherent loads
                  aq[q] = cn > 0 ? __ldcg(reinterpret_cast<const uint4*>(y0r + col0) + q) : z4;
                  bq[q] = cn > 1 ? __ldcg(reinterpret_cast<const uint4*>(y1r + col0) + q) : z4;
                }
                const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(xq);
                const __nv_bfloat16* ab = reinterpret_cast<const __nv_bfloat16*>(aq);
                const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(bq);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  float acc_m = 0.f;  // the zero accumulator of scatter_rows
                  if (cn > 0) acc_m = __fadd_rn(acc_m, __fmul_rn(cp0, __bfloat162float(ab[i])));
                  if (cn > 1) acc_m = __fadd_rn(acc_m, __fmul_rn(cp1, __bfloat162float(bb[i])));
                  v[i] = __fadd_rn(__fadd_rn(__bfloat162float(xb[i]), acc_m), v[i]);
                }
                uint4* dst = reinterpret_cast<uint4*>(drow + col0);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  uint4 pk;
                  pk.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                  pk.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                  pk.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                  pk.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                  if (args.stream_hint)
                    st_global_hint(dst + q, pk, pol_stream);
                  else
                    dst[q] = pk;
                }
              } else {
                for (int i = 0; i < 32; ++i) {
                  if (col0 + i >= N) break;
                  float acc_m = 0.f;
                  if (cn > 0) acc_m = __fadd_rn(acc_m, __fmul_rn(cp0, __bfloat162float(__ldcg(y0r + col0 + i))));
                  if (cn > 1) acc_m = __fadd_rn(acc_m, __fmul_rn(cp1, __bfloat162float(__ldcg(y1r + col0 + i))));
                  drow[col0 + i] = __float2bfloat16_rn(
                      __fadd_rn(__fadd_rn(__bfloat162float(xrow[col0 + i]), acc_m), v[i]));
                }
              }
              continue;
            }
          }
          if constexpr (EPI == EPI_WGRAD_ACC) {  // split-K partial: fp32 reduction in HBM/L2
            if (kzero) continue;
            float* dst = args.Dacc + out_row * N + col0;
            if ((N % 4) == 0 && col0 + 32 <= N) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                red_add_v4_f32(dst + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i < N) atomicAdd(dst + i, v[i]);
            }
            continue;
          }
          if constexpr (EPI == EPI_WGRAD) {
            if (kzero) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.f;
            }
          }
          if constexpr (EPI == EPI_GELU_SAVE) {
            if (vec_ok && col0 + 32 <= N) {
              uint4* ad = reinterpret_cast<uint4*>(arow + col0);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                uint4 pk;
                pk.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                pk.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                pk.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                pk.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                ad[q] = pk;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i < N) arow[col0 + i] = __float2bfloat16_rn(v[i]);
            }
          }
          if constexpr (EPI == EPI_BIAS_GELU) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = gelu_tanh_fast_half(v[i]);
          }
          if constexpr (EPI == EPI_GELU_SAVE) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = gelu_tanh_fast(v[i]);
          }
          if constexpr (EPI == EPI_GELU_BWD) {  // no bias: D = dH, times gelu'(a)
            if (vec_ok && col0 + 32 <= N) {
              const __nv_bfloat16* ab = reinterpret_cast<const __nv_bfloat16*>(xbuf[xslot(c)]);
#pragma unroll
              for (int i = 0; i < 32; ++i)
                v[i] = __uint_as_float(r[c % kRB][i]) * gelu_tanh_grad_fast(__bfloat162float(ab[i]));
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i < N)
                  v[i] = __uint_as_float(r[c % kRB][i]) *
                         gelu_tanh_grad_fast(__bfloat162float(xrow[col0 + i]));
            }
          }
          if constexpr (is_combine<EPI>()) {
            // training: also keep y = acc + b2 (row layout) for backward (valid rows
            // only: with coalesced stores every lane of the warp reaches this point, and
            // a tile's rows past the group's count may lie in the next group's block)
            if (args.D != nullptr && valid) {
              __nv_bfloat16* yrow = args.D + out_row * N;
              if (vec_ok && col0 + 32 <= N) {
                uint4* yd = reinterpret_cast<uint4*>(yrow + col0);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  uint4 pk;
                  pk.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                  pk.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                  pk.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                  pk.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                  yd[q] = pk;
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (col0 + i < N) yrow[col0 + i] = __float2bfloat16_rn(v[i]);
              }
            }
            if (vec_ok && col0 + 32 <= N) {
              const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(xbuf[xslot(c)]);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = fmaf(prob, v[i], __bfloat162float(xb[i]));
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i < N) v[i] = fmaf(prob, v[i], __bfloat162float(xrow[col0 + i]));
            }
          }
          if constexpr (kTmaEpi) {
            if (args.tma_store) {
              uint32_t pk32[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) pk32[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
              stage_store(pk32);
              continue;
            }
          }
          if constexpr (kCoalOK) {
            if (coal) {  // warp-uniform: every lane of the warp is here (invalid rows masked)
              uint8_t* ob = smem + L::kOutOff + (warp - 2) * (out_stage_bytes<EPI, EW, CG, BN>() / EW);
              __syncwarp();
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int chunk = q ^ ((lane >> 1) & 3);
                *reinterpret_cast<uint4*>(ob + lane * 64 + chunk * 16) =
                    make_uint4(pack_bf16x2(v[8 * q + 0], v[8 * q + 1]),
                               pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                               pack_bf16x2(v[8 * q + 4], v[8 * q + 5]),
                               pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
              }
              __syncwarp();
              const unsigned long long mine =
                  valid ? reinterpret_cast<unsigned long long>(drow + col0) : 0ull;
#pragma unroll
              for (int it = 0; it < 4; ++it) {
                const int r = it * 8 + (int)(lane >> 2), part = lane & 3;
                const unsigned long long dst = __shfl_sync(0xffffffffu, mine, r);
                const uint4 val =
                    *reinterpret_cast<const uint4*>(ob + r * 64 + ((part ^ ((r >> 1) & 3)) * 16));
                if (dst) reinterpret_cast<uint4*>(dst)[part] = val;
              }
              __syncwarp();
              continue;
            }
          }
          if (vec_ok && col0 + 32 <= N) {
            uint4* dst = reinterpret_cast<uint4*>(drow + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 pk;
              pk.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
              pk.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
              pk.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
              pk.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
              if (args.stream_hint && !push)
                st_global_hint(dst + q, pk, pol_stream);
              else
                dst[q] = pk;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < N) drow[col0 + i] = __float2bfloat16_rn(v[i]);
          }
        }
        if constexpr (!kSplit) {  // (kSplit handed every part back as it was read)
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2)
              mbar_arrive_cluster(&tempty[acc], pl);  // the leader's MMA reuses it
            else
              mbar_arrive(&tempty[acc]);
          }
        }
        if constexpr (EPI == EPI_BIAS_RESID) {
          if (args.has_rc && !rc) {
            // expert tile: publish this warp's y stores to the shared-MLP epilogues
            // (bulk TMA stores complete -> async-proxy writes ordered before the release)
            __threadfence();
            __syncwarp();
            if (lane == 0) {
              bulk_wait_group_all();
              fence_proxy_async_global();
              red_release_gpu_add(args.c_done, 1);
            }
            __syncwarp();
          }
        }
      } else {
        // ---------------- gate epilogue: thread = token row, BN >= E columns
        const int E = args.E;
        // MS > 1: sub-tile ms = the pair tile ms*TM rows further, its accumulator
        // ms*BN TMEM columns further (both sub-tiles shared every W_g^T stage)
        for (int ms = 0; ms < MS; ++ms) {
        const uint32_t t_addr = t_addr0 + ms * BN;
        const int64_t t = out_row + ms * TM;  // single group: rows are tokens
        const bool valid = local_row + ms * TM < rows_g && !g_skip;
        float b1 = -INFINITY, b2 = -INFINITY;
        int i1 = 0x7fffffff, i2 = 0x7fffffff;
        // top-k scan; K1: the arg-max alone (k = 1: 3 instructions per logit, not 8), as
        // four interleaved chains (columns i mod 4, each ascending with a strict compare,
        // merged below preferring the lower index on equal values) so the dependent
        // select chain is a quarter as long
        float pb[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        int pi[4] = {0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff};
        auto topk_scan = [&](auto k1) {
          constexpr bool K1 = decltype(k1)::value;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_addr + c * 32, r);
            tmem_ld_wait();
            // ascending column order + strict compare keeps the lower index on ties
            // (branch-free selects; padded columns >= E are masked to -inf)
            const bool full_chunk = c * 32 + 32 <= E;
            // K1: chunk-local chains whose index is the compile-time column in the
            // chunk (a select of an immediate), folded into pb / pi after the chunk
            float qb[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
            int qi[4] = {0, 0, 0, 0};
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int col = c * 32 + i;
              const float v = (full_chunk || col < E) ? __uint_as_float(r[i]) : -INFINITY;
              if constexpr (K1) {
                const bool g = v > qb[i & 3];
                qb[i & 3] = g ? v : qb[i & 3];
                qi[i & 3] = g ? i : qi[i & 3];
              } else {
                const bool g1 = v > b1, g2 = v > b2;
                b2 = g1 ? b1 : (g2 ? v : b2);
                i2 = g1 ? i1 : (g2 ? col : i2);
                b1 = g1 ? v : b1;
                i1 = g1 ? col : i1;
              }
            }
            if constexpr (K1) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {  // later chunks hold higher columns: strict >
                const bool g = qb[j] > pb[j];
                pb[j] = g ? qb[j] : pb[j];
                pi[j] = g ? c * 32 + qi[j] : pi[j];
              }
            }
            if (valid && args.logits != nullptr) {
              float* lrow = args.logits + t * E;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c * 32 + i < E) lrow[c * 32 + i] = __uint_as_float(r[i]);
            }
          }
        };
        if (args.k == 1) {
          topk_scan(std::true_type{});
          if (warp == 2 && lane == 0 && vit == 0) GATE_TRACE(9);
#pragma unroll
          for (int j = 0; j < 4; ++j) {  // merge: larger value, then lower index
            const bool g = pb[j] > b1 || (pb[j] == b1 && pi[j] < i1);
            b1 = g ? pb[j] : b1;
            i1 = g ? pi[j] : i1;
          }
        } else {
          topk_scan(std::false_type{});
        }
        // Rows with fewer than k values above -inf (NaN / -inf logits, e.g. after a
        // diverged step) re-rank with np.argsort(-logits, kind="stable") semantics:
        // NaN after every number, -inf before NaN, ties to the lower index - so
        // every id stays inside [0, E). Warp-uniform (tcgen05.ld is collective).
        const bool slow = i1 == 0x7fffffff || (args.k == 2 && i2 == 0x7fffffff);
        if (__any_sync(0xffffffffu, slow)) {
          float s1 = 0.f, s2 = 0.f;
          int j1 = -1, j2 = -1;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_addr + c * 32, r);
            tmem_ld_wait();
#pragma unroll 1
            for (int i = 0; i < 32; ++i) {
              const int col = c * 32 + i;
              if (col >= E) break;
              const float v = __uint_as_float(r[i]);
              const bool vn = v != v;
              const bool g1 = j1 < 0 || (!vn && ((s1 != s1) || v > s1));
              const bool g2 = !g1 && (j2 < 0 || (!vn && ((s2 != s2) || v > s2)));
              if (g1) { s2 = s1; j2 = j1; s1 = v; j1 = col; }
              else if (g2) { s2 = v; j2 = col; }
            }
          }
          if (slow) { b1 = s1; i1 = j1; b2 = s2; i2 = j2; }
        }
        // softmax denominator: exp(v - b1) = 2^(v*log2e - b1*log2e) on the MUFU (one FFMA +
        // one EX2 per logit; +-inf / NaN rows give the same inf / NaN / 0 terms as expf)
        float sum = 0.f;
        const float nb1 = -b1 * kLog2e;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(t_addr + c * 32, r);
          tmem_ld_wait();
          if (c * 32 + 32 <= E) {
            float ps[4] = {0.f, 0.f, 0.f, 0.f};  // four partial sums: a quarter-length FADD chain
#pragma unroll
            for (int i = 0; i < 32; ++i) ps[i & 3] += ex2_approx(fmaf(__uint_as_float(r[i]), kLog2e, nb1));
            sum += (ps[0] + ps[1]) + (ps[2] + ps[3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i < E) sum += ex2_approx(fmaf(__uint_as_float(r[i]), kLog2e, nb1));
          }
        }
        if (warp == 2 && lane == 0 && vit == 0) GATE_TRACE(10);
        if (args.probsum != nullptr) {
          // load-balance statistics (arch.py:297-313): column sums of the full softmax,
          // reduced across the warp with a transpose-reduce (lane l ends with column l)
          const float inv = 1.f / sum;
          float* psum = reinterpret_cast<float*>(smem + L::kTileOff) + 8 + 4 * E;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_addr + c * 32, r);
            tmem_ld_wait();
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i)
              v[i] = (valid && c * 32 + i < E) ? expf(__uint_as_float(r[i]) - b1) * inv : 0.f;
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
              const bool upper = (lane & off) != 0;
#pragma unroll
              for (int i = 0; i < off; ++i) {
                const float send = upper ? v[i] : v[i + off];
                const float keep = upper ? v[i + off] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
              }
            }
            if (c * 32 + (int)lane < E) atomicAdd(&psum[c * 32 + lane], v[0]);
          }
        }
        // accumulator consumed: hand TMEM back to the MMA warp (the leader's, CG=2)
        tc_fence_before();
        __syncwarp();
        if (lane == 0 && ms == MS - 1) {
          if constexpr (CG == 2)
            mbar_arrive_cluster(&tempty[acc], pl);
          else
            mbar_arrive(&tempty[acc]);
        }

        const int k = args.k;
        int e0 = valid ? i1 : -1;
        int e1 = (valid && k == 2) ? i2 : -2;
        if (valid) {
          args.ids[t * k] = i1;
          args.gate_probs[t * k] = 1.0f / sum;  // exp(b1 - b1) / sum
          if (k == 2) {
            args.ids[t * k + 1] = i2;
            args.gate_probs[t * k + 1] = expf(b2 - b1) / sum;
          }
        }
        if (warp == 2 && lane == 0 && vit == 0) GATE_TRACE(11);
        // per-tile capacity ranks (token-major order, gating.py:226)
        // 4 x E per-warp counters in the tile-table region (G == 1 uses [0, 2))
        int* wc = reinterpret_cast<int*>(smem + L::kTileOff) + 8;
        const int tid = (warp - 2) * 32 + lane;  // 0..127
        for (int i = tid; i < 4 * E; i += 128) wc[i] = 0;
        named_bar_sync(1, 128);
        int r0 = 0, r1 = 0;
        if (k == 1) {
          unsigned m = __match_any_sync(0xffffffffu, e0);
          r0 = __popc(m & ((1u << lane) - 1u));
        } else {
          for (int l = 0; l < 32; ++l) {
            int o0 = __shfl_sync(0xffffffffu, e0, l);
            int o1 = __shfl_sync(0xffffffffu, e1, l);
            if (l < (int)lane) {
              r0 += (o0 == e0) + (o1 == e0);
              r1 += (o0 == e1) + (o1 == e1);
            }
          }
        }
        if (valid) {
          atomicAdd(&wc[quarter * E + e0], 1);
          if (k == 2) atomicAdd(&wc[quarter * E + e1], 1);
        }
        named_bar_sync(1, 128);
        if (valid) {
          for (uint32_t q = 0; q < quarter; ++q) {
            r0 += wc[q * E + e0];
            if (k == 2) r1 += wc[q * E + e1];
          }
          args.local_rank[t * k] = r0;
          if (k == 2) args.local_rank[t * k + 1] = r1;
        }
        if (warp == 2 && lane == 0 && vit == 0) GATE_TRACE(12);
        const int64_t tile_row0 = gbal ? (int64_t)tile * BM + cta * BM
                                       : (int64_t)mb * TMC + pair * TM + ms * TM + cta * BM;  // this CTA's routing tile
        if (tile_row0 < args.S && !g_skip)
          for (int e = tid; e < E; e += 128)
            args.tile_counts[tile_row0 / kRouteTile * E + e] =
                wc[e] + wc[E + e] + wc[2 * E + e] + wc[3 * E + e];
        named_bar_sync(1, 128);
        }  // ms
        if (warp == 2 && lane == 0 && vit == 0) GATE_TRACE(6);
      }
      if (++acc == AS) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (EPI == EPI_WGRAD || args.tma_store) {
      if (lane == 0) bulk_wait_group_all();
      __syncwarp();
    }
    // pushed rows (NVLink stores to the sources) performed before the kernel ends
    // and the caller's flag barrier releases them
    if (args.push_base != nullptr) __threadfence_system();
    if constexpr (EPI == EPI_GATE) {
      if (args.probsum != nullptr) {  // one global atomic per expert per CTA
        named_bar_sync(1, 128);
        const float* psum = reinterpret_cast<const float*>(smem + L::kTileOff) + 8 + 4 * args.E;
        for (int i = (warp - 2) * 32 + lane; i < args.E; i += 128) atomicAdd(&args.probsum[i], psum[i]);
      }
    }
  } else if constexpr (kMN) {
    // ===================== fix-up warp (weight gradients): walks the producer's
    // stage sequence; for each partial K block waits for its TMA, zeroes the rows
    // >= rem (whole 128-B lines: the swizzle only permutes chunks inside a line),
    // makes the writes visible to the tensor core and releases the stage
    int stage = 0;
    uint32_t pph = 0;  // per-stage parity of pbar
    int g = 0;
    constexpr int kBoxB = (BN / CG) / 64;
    for (int it = 0;; ++it) {
      const int tile = fetch(it, false);
      if (tile < 0) break;
      int mb, nb;
      decode(tile, g, mb, nb);
      const int kg = (int)(args.k_rows ? args.k_rows[g] : args.k_rows_const);
      const int kb_end = (kg + BK - 1) / BK;
      if (kb_end > 0) {
        stage = (stage + kb_end - 1) % STAGES;  // only the last K block can be partial
        const int rem = kg - (kb_end - 1) * BK;
        if (rem < BK) {
          mbar_wait(&pbar[stage], (pph >> stage) & 1u);
          pph ^= 1u << stage;
          uint8_t* sa = smem + stage * L::kStageBytes;
          const uint4 z = make_uint4(0u, 0u, 0u, 0u);
          for (int box = 0; box < 2 + kBoxB; ++box) {  // A's 2 boxes, then B's
            uint4* base = reinterpret_cast<uint4*>(sa + box * 8192);
            for (int i = rem * 8 + (int)lane; i < 512; i += 32) base[i] = z;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) {
              if (leader)
                mbar_arrive(&full[stage]);
              else
                mbar_arrive_cluster_release(&full[stage], pl);
            } else {
              mbar_arrive(&full[stage]);
            }
          }
          __syncwarp();
        }
        stage = (stage + 1) % STAGES;
      }
    }
  }

  if (threadIdx.x == 0) GATE_TRACE(7);
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();  // the peer's TMEM is written by the leader's MMAs: free only when both done
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc_cg2(tmem_base, tmem_cols<BN, MS>());
    else
      tmem_dealloc(tmem_base, tmem_cols<BN, MS>());
  }
  if (threadIdx.x == 0) GATE_TRACE(8);
}

// ============================================================ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 row-major [rows, cols] tensor map, box [box_rows, 64 cols], 128B swizzle.
static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) return MOE_ENODRV;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : MOE_ETMA;
}

// 3-D bf16 [G][P][N] output map for the weight-gradient TMA stores: box 32 x 32 x 1,
// 64-B swizzle (matches the epilogue's staging layout); clips at P and N.
static int make_map_out3d(CUtensorMap* map, void* base, int64_t G, int64_t P, int64_t N) {
  auto enc = get_encode();
  if (!enc) return MOE_ENODRV;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)P, (cuuint64_t)G};
  cuuint64_t strides[2] = {(cuuint64_t)(N * 2), (cuuint64_t)(P * N * 2)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : MOE_ETMA;
}

// MOE_PREFETCH bit 0: gate GEMM prefetches the next tile's x; bit 1: expert
// GEMMs prefetch the next tile's weights. Tuning knob, default off: measured on
// B200 the gate did not speed up and the expert GEMMs slowed by 10-30%.
static int prefetch_mode() {
  static const int m = [] {
    const char* v = getenv("MOE_PREFETCH");
    return v ? atoi(v) : 0;
  }();
  return m;
}

// Dynamic-scheduling tile counters: a per-device pool, one zeroed (stream-ordered
// memset) slot per launch, rotating so launches in flight on other streams do not
// share a counter. MOE_DYN_SCHED=0 restores static round robin.
// mode 2 (default): only long-K launches (K >= 2N, the GEMM2 shape: few long
// tiles, where keeping the weight-sharing pairs in step pays: GEMM2 1.65 vs
// 1.70 ms in the C3 layer); 1: every launch (GEMM1, 4x more and shorter tiles,
// loses 2-4% to the queue hand-off); 0: static round robin everywhere.
static int* dyn_counter(cudaStream_t st, int64_t K = 0, int64_t N = 0, bool force = false) {
  static const int enabled = [] {
    const char* v = getenv("MOE_DYN_SCHED");
    return v ? atoi(v) : 2;
  }();
  if (!force && (!enabled || (enabled == 2 && K < 2 * N))) return nullptr;
  // slots [0, kPool) rotate for eager launches; launches captured into CUDA graphs
  // take slots from [kPool, 2*kPool) that are never handed out again (a replayed
  // graph re-zeroes and reuses its own slot), static schedule once those run out
  constexpr int kPool = 4096;
  static int* pool[64] = {};
  static unsigned next[64] = {}, next_graph[64] = {};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  int* c = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (pool[dev] == nullptr) {
      if (capturing) return nullptr;  // no allocation inside a capture
      if (cudaMalloc(&pool[dev], 2 * kPool * sizeof(int)) != cudaSuccess) {
        pool[dev] = nullptr;
        return nullptr;
      }
    }
    if (capturing) {
      if (next_graph[dev] >= (unsigned)kPool) return nullptr;
      c = pool[dev] + kPool + next_graph[dev]++;
    } else {
      c = pool[dev] + (next[dev]++ % kPool);
    }
  }
  if (cudaMemsetAsync(c, 0, sizeof(int), st) != cudaSuccess) return nullptr;
  return c;
}

// A per-device side stream + fork/join events for the hybrid GEMM launch.
static bool side_stream(cudaStream_t* s, cudaEvent_t* fork, cudaEvent_t* join) {
  static cudaStream_t streams[64] = {};
  static cudaEvent_t forks[64] = {}, joins[64] = {};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  std::lock_guard<std::mutex> lock(mu);
  if (streams[dev] == nullptr) {
    if (cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&forks[dev], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&joins[dev], cudaEventDisableTiming) != cudaSuccess)
      return false;
  }
  *s = streams[dev];
  *fork = forks[dev];
  *join = joins[dev];
  return true;
}

// Per-device launch facts, cached per device ordinal (the library targets the
// current device; one process may drive several GPUs, from several threads).
constexpr int kMaxDevices = 64;

static int cur_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return -1;
  return dev;
}

static int num_sms() {
  static std::atomic<int> n[kMaxDevices];
  const int dev = cur_device();
  if (dev < 0) return 148;
  int v = n[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1)
      v = 148;
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) binds to the current device's
// context: set it once per (kernel instance, device). Setting it twice is benign,
// so concurrent first calls only race to do the same work.
template <typename Kern>
static cudaError_t ensure_smem_attr(Kern kern, int bytes, std::atomic<uint64_t>& done_mask) {
  const int dev = cur_device();
  if (dev < 0) return cudaErrorInvalidDevice;
  const uint64_t bit = 1ull << dev;
  if (done_mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done_mask.fetch_or(bit, std::memory_order_release);
  return e;
}

template <int BN, int STAGES, int EPI, int CG = 1, int EW = 4, int CL = CG, int SUB = 1,
          int MS = 1>
static int launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& args,
                     int64_t max_tiles, cudaStream_t st, const CUtensorMap* md = nullptr,
                     int64_t grid_cap = 0, const CUtensorMap* ma2 = nullptr, int ctas_per_sm = 1) {
  using L = Smem<BN, STAGES, CG, out_stage_bytes<EPI, EW, CG, BN>(), MS>;
  static_assert(L::kTotal <= 227 * 1024, "dynamic shared memory beyond the 227 KB per CTA");
  auto kern = gemm_bf16_tc_kernel<BN, STAGES, EPI, CG, EW, CL, SUB, MS>;
  static std::atomic<uint64_t> attr_done{0};
  {
    cudaError_t e = ensure_smem_attr(kern, L::kTotal, attr_done);
    if (e != cudaSuccess) return (int)e;
  }
  int64_t grid = (int64_t)num_sms() * ctas_per_sm;
  if (gemm_cta_limit() > 0 && gemm_cta_limit() < grid) grid = gemm_cta_limit();
  if (grid_cap > 0 && grid_cap < grid) grid = grid_cap;
  // max_tiles counts cluster tiles (CL/CG pairs each)
  if (max_tiles * CL < grid) grid = max_tiles < 1 ? CL : max_tiles * CL;
  grid -= grid % CL;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(threads_for<EW, EPI>());
  cfg.dynamicSmemBytes = L::kTotal;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  if constexpr (CL > 2) {
    // 4-CTA clusters must fit whole GPCs: size the persistent grid to what can be resident
    static std::atomic<int> clusters_by_dev[kMaxDevices];
    const int dev = cur_device();
    int max_clusters = dev >= 0 ? clusters_by_dev[dev].load(std::memory_order_relaxed) : 0;
    if (max_clusters == 0) {
      if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess ||
          max_clusters < 1)
        max_clusters = (int)(num_sms() / CL);
      if (dev >= 0) clusters_by_dev[dev].store(max_clusters, std::memory_order_relaxed);
    }
    if (grid > (int64_t)max_clusters * CL) grid = (int64_t)max_clusters * CL;
    cfg.gridDim = dim3((unsigned)grid);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, md ? *md : mb, args, ma2 ? *ma2 : ma);
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

// Resident 4-CTA clusters of the forward GEMM (B200: 33 -> 132 of 148 SMs).
static int max_clusters4(bool gelu) {
  static std::atomic<int> n[kMaxDevices][2];
  const int dev = cur_device();
  if (dev < 0) return num_sms() / 4;
  int v = n[dev][gelu ? 1 : 0].load(std::memory_order_relaxed);
  if (v == 0) {
    using L = Smem<256, 5, 2, out_stage_bytes<EPI_BIAS, 8, 2, 256>()>;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(4 * 64);
    cfg.blockDim = dim3(threads_for<8, EPI_BIAS>());
    cfg.dynamicSmemBytes = L::kTotal;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 4;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto kern = gelu ? gemm_bf16_tc_kernel<256, 5, EPI_BIAS_GELU, 2, 8, 4>
                     : gemm_bf16_tc_kernel<256, 5, EPI_BIAS, 2, 8, 4>;
    static std::atomic<uint64_t> attr_done[2];
    ensure_smem_attr(kern, L::kTotal, attr_done[gelu ? 1 : 0]);
    if (cudaOccupancyMaxActiveClusters(&v, kern, &cfg) != cudaSuccess || v < 1)
      v = num_sms() / 4;
    n[dev][gelu ? 1 : 0].store(v, std::memory_order_relaxed);
  }
  return v;
}

int launch_grouped_gemm_bf16(const void* A, int64_t a_rows, int K, const void* B, int64_t b_rows,
                             int N, const float* bias, void* D, int G, const int32_t* row_start,
                             int64_t row_stride, const int32_t* rows, int64_t rows_const,
                             const int32_t* weight_idx, int64_t max_group_rows, int act,
                             cudaStream_t st, const int32_t* row_token, const float* row_prob,
                             const void* x_resid, void* out, int x_by_row, int pad_scratch,
                             const int32_t* a_gather, void* const* push_base,
                             const int32_t* row_src) {
  if (G < 1 || G > kMaxGroups || K < 1 || N < 1 || (K % 8) != 0) return MOE_EINVAL;
  const bool force256 = (pad_scratch & 2) != 0;  // MOE_GEMM_TILE256
  pad_scratch &= 1;
  int BN = 256;
  if (N <= 32) BN = 32;
  else if (N <= 64) BN = 64;
  else if (N <= 128) BN = 128;
  // 2-CTA 256x256 tiles for the big expert GEMMs; 1-CTA 128-row tiles when groups are
  // small (decode) or N is narrow
  // MOE_GEMM_VARIANT (tuning knob, default 0): 0 = 2-CTA + 8 epilogue warps,
  // 1 = 2-CTA + 4 epilogue warps, 2 = 1-CTA + 4 epilogue warps
  static const int variant = [] {
    const char* v = getenv("MOE_GEMM_VARIANT");
    return v ? atoi(v) : 0;
  }();
  static const int stream_hint = [] {
    const char* v = getenv("MOE_STORE_HINT");
    return v ? atoi(v) : 1;
  }();
  static const int raster = [] {
    const char* v = getenv("MOE_RASTER");
    return v ? atoi(v) : 0;
  }();
  const int CG = (BN == 256 && max_group_rows > BM && variant != 2) ? 2 : 1;
  CUtensorMap ma, mb;
  // gather mode: A is the token matrix X (a_rows rows), one 128-B box row per gather lane
  int rc = make_map(&ma, A, a_rows, K, a_gather ? 1 : BM);
  if (rc) return rc;
  rc = make_map(&mb, B, b_rows, K, BN / CG);
  if (rc) return rc;
  GemmArgs a{};
  a.bias = bias;
  a.D = (__nv_bfloat16*)D;
  a.K = K;
  a.N = N;
  a.G = G;
  a.row_start = row_start;
  a.row_stride = row_stride;
  a.rows = rows;
  a.rows_const = rows_const;
  a.weight_idx = weight_idx;
  a.row_token = row_token;
  a.row_prob = row_prob;
  a.x_resid = (const __nv_bfloat16*)x_resid;
  a.out = (__nv_bfloat16*)out;
  a.x_by_row = x_by_row;
  a.a_gather = a_gather;
  a.push_base = push_base;
  a.row_src = row_src;
  static const int coal = [] {  // MOE_COMBINE_COAL (default 1): coalesced combine stores
    const char* v = getenv("MOE_COMBINE_COAL");
    return v ? atoi(v) : 1;
  }();
  a.coal_store = coal;
  a.tile_counter = dyn_counter(st, K, N);
  a.stream_hint = stream_hint;
  a.raster = raster;
  a.prefetch = prefetch_mode() & 2 ? 1 : 0;
  const int64_t nblk = (N + BN - 1) / BN;
  const int64_t tm = (int64_t)BM * CG;
  const int64_t max_tiles = (int64_t)G * ((max_group_rows + tm - 1) / tm) * nblk;
  if (max_tiles == 0) return 0;
  const bool gelu = act == 1;
  if (act == 3 || act == 4) {  // training: GELU saving the pre-activation / GELU backward
    const bool save = act == 3;
    if (CG == 2)
      return save ? launch_tc<256, 6, EPI_GELU_SAVE, 2, 8>(ma, mb, a, max_tiles, st)
                  : launch_tc<256, 6, EPI_GELU_BWD, 2, 8>(ma, mb, a, max_tiles, st);
    switch (BN) {
      case 32:
        return save ? launch_tc<32, 8, EPI_GELU_SAVE, 1, 4>(ma, mb, a, max_tiles, st)
                    : launch_tc<32, 8, EPI_GELU_BWD, 1, 4>(ma, mb, a, max_tiles, st);
      case 64:
        return save ? launch_tc<64, 8, EPI_GELU_SAVE, 1, 8>(ma, mb, a, max_tiles, st)
                    : launch_tc<64, 8, EPI_GELU_BWD, 1, 8>(ma, mb, a, max_tiles, st);
      case 128:
        return save ? launch_tc<128, 6, EPI_GELU_SAVE, 1, 8>(ma, mb, a, max_tiles, st)
                    : launch_tc<128, 6, EPI_GELU_BWD, 1, 8>(ma, mb, a, max_tiles, st);
      default:
        return save ? launch_tc<256, 4, EPI_GELU_SAVE, 1, 4>(ma, mb, a, max_tiles, st)
                    : launch_tc<256, 4, EPI_GELU_BWD, 1, 4>(ma, mb, a, max_tiles, st);
    }
  }
  if (act == 2) {  // fused combine epilogue
    // 256 x 512 fused-combine tiles (MOE_COMBINE_BN512=1): the epilogue streams
    // chunk by chunk (kStream), 25% fewer operand bytes per flop than 256 x 256
    static const int bn512c = [] {
      const char* v = getenv("MOE_COMBINE_BN512");
      return v ? atoi(v) : 0;
    }();
    if (CG == 2 && bn512c == 1 && push_base == nullptr && (N % 512) == 0) {
      CUtensorMap mb2;
      rc = make_map(&mb2, B, b_rows, K, 128);
      if (rc) return rc;
      const int64_t tiles512 = (int64_t)G * ((max_group_rows + tm - 1) / tm) * ((N + 511) / 512);
      return launch_tc<512, 4, EPI_BIAS_COMBINE, 2, 8>(ma, mb2, a, tiles512, st);
    }
    if (CG == 2)
      return push_base ? launch_tc<256, 6, EPI_COMBINE_PUSH, 2, 8>(ma, mb, a, max_tiles, st)
                       : launch_tc<256, 6, EPI_BIAS_COMBINE, 2, 8>(ma, mb, a, max_tiles, st);
    if (push_base != nullptr) {  // EP push return on 1-CTA tiles (small groups)
      switch (BN) {
        case 32: return launch_tc<32, 8, EPI_COMBINE_PUSH, 1, 4>(ma, mb, a, max_tiles, st);
        case 64: return launch_tc<64, 8, EPI_COMBINE_PUSH, 1, 8>(ma, mb, a, max_tiles, st);
        case 128: return launch_tc<128, 6, EPI_COMBINE_PUSH, 1, 8>(ma, mb, a, max_tiles, st);
        default: return launch_tc<256, 4, EPI_COMBINE_PUSH, 1, 4>(ma, mb, a, max_tiles, st);
      }
    }
    switch (BN) {
      case 32: return launch_tc<32, 8, EPI_BIAS_COMBINE, 1, 4>(ma, mb, a, max_tiles, st);
      case 64: return launch_tc<64, 8, EPI_BIAS_COMBINE, 1, 8>(ma, mb, a, max_tiles, st);
      case 128: return launch_tc<128, 6, EPI_BIAS_COMBINE, 1, 8>(ma, mb, a, max_tiles, st);
      default: return launch_tc<256, 4, EPI_BIAS_COMBINE, 1, 4>(ma, mb, a, max_tiles, st);
    }
  }
  if (CG == 2 && variant == 1)
    return gelu ? launch_tc<256, 6, EPI_BIAS_GELU, 2, 4>(ma, mb, a, max_tiles, st)
                : launch_tc<256, 6, EPI_BIAS, 2, 4>(ma, mb, a, max_tiles, st);
  if (CG == 2) {
    // whole-box TMA stores when the groups' padding rows are scratch (strided groups)
    CUtensorMap md;
    const int64_t per_group = row_stride > 0 ? row_stride : (G == 1 ? rows_const : 0);
    static const int tma_epi = [] {
      const char* v = getenv("MOE_TMA_EPILOGUE");
      return v ? atoi(v) : 1;
    }();
#ifndef MOE_FWD_STAGES
#define MOE_FWD_STAGES 5
#endif
#ifndef MOE_FWD_EW
#define MOE_FWD_EW 8
#endif
    // MOE_BN512: 256 x 512 pair tiles (25% less operand traffic per flop) for
    // 0 none, 1 every eligible forward GEMM incl. the fused combine, 2 the
    // plain-bias ones, 3 (default) plain-bias + bias/GELU launches of >= 1 TFLOP.
    // Measured: plain-bias C2 / C4 +3-5%; GEMM1 (GELU, its epilogue staging each
    // accumulator half in registers) wins only where the launch is long enough to
    // run at the 1 kW cap, where operand traffic is energy (C3: layer +1%, GEMM1
    // up to -4%), and loses 5-10% at full clock (C2 / C4 GEMM1); the fused combine
    // is 2% slower on it (mode 1 only)
    static const int bn512 = [] {
      const char* v = getenv("MOE_BN512");
      return v ? atoi(v) : 3;
    }();
    const bool long_launch = 2.0 * (double)G * (double)max_group_rows * N * K >= 1e12;
    static const int cluster4 = [] {
      const char* v = getenv("MOE_CLUSTER4");
      return v ? atoi(v) : 0;
    }();
    if (!force256 && (bn512 == 1 || (bn512 >= 2 && !gelu) || (bn512 == 3 && long_launch)) && tma_epi && pad_scratch && row_start == nullptr && per_group > 0 &&
        (N % 512) == 0 && make_map_out3d(&md, D, G, per_group, N) == 0) {
      // 256 x 512 pair tiles; TMEM holds one accumulator, handed over in two halves
      CUtensorMap mb2;
      if ((cluster4 == 3 || cluster4 == 4) && a_gather == nullptr) {
        // MOE_CLUSTER4=3: two such pairs per 4-CTA cluster sharing the weight tile
        // by multicast (512 x 512 per cluster; only whole-GPC clusters fit: 33 of
        // them, 132 SMs). =4: plus a 2-CTA instance on the SMs they leave (each
        // pair runs both 256-row halves of a 512 x 512 tile), both instances
        // pulling tiles from one dynamic counter on two streams
        CUtensorMap mb64;
        rc = make_map(&mb64, B, b_rows, K, 64);
        if (rc) return rc;
        a.tma_store = 1;
        const int64_t tiles4 = (int64_t)G * ((max_group_rows + 2 * tm - 1) / (2 * tm)) * ((N + 511) / 512);
        const int nclus = max_clusters4(gelu);
        const int64_t left = num_sms() - 4 * (int64_t)nclus;
        int* ctr = cluster4 == 4 ? dyn_counter(st, 0, 0, true) : nullptr;
        if (ctr == nullptr || left < 2) {
          a.tile_counter = nullptr;  // the pairs of a cluster move in step (static schedule)
          return gelu ? launch_tc<512, 4, EPI_BIAS_GELU, 2, 8, 4>(ma, mb64, a, tiles4, st, &md)
                      : launch_tc<512, 4, EPI_BIAS, 2, 8, 4>(ma, mb64, a, tiles4, st, &md);
        }
        rc = make_map(&mb2, B, b_rows, K, 128);
        if (rc) return rc;
        a.tile_counter = ctr;
        cudaStream_t side;
        cudaEvent_t fork, join;
        if (!side_stream(&side, &fork, &join)) return MOE_EINVAL;
        cudaEventRecord(fork, st);
        cudaStreamWaitEvent(side, fork, 0);
        int r1 = gelu ? launch_tc<512, 4, EPI_BIAS_GELU, 2, 8, 4>(ma, mb64, a, tiles4, st, &md)
                      : launch_tc<512, 4, EPI_BIAS, 2, 8, 4>(ma, mb64, a, tiles4, st, &md);
        int r2 = gelu ? launch_tc<512, 4, EPI_BIAS_GELU, 2, 8, 2, 2>(ma, mb2, a, tiles4, side, &md,
                                                                       left - left % 2)
                      : launch_tc<512, 4, EPI_BIAS, 2, 8, 2, 2>(ma, mb2, a, tiles4, side, &md,
                                                               left - left % 2);
        cudaEventRecord(join, side);
        cudaStreamWaitEvent(st, join, 0);
        return r1 ? r1 : r2;
      }
      rc = make_map(&mb2, B, b_rows, K, 128);
      if (rc) return rc;
      a.tma_store = 1;
      const int64_t tiles512 = (int64_t)G * ((max_group_rows + tm - 1) / tm) * ((N + 511) / 512);
      return gelu ? launch_tc<512, 4, EPI_BIAS_GELU, 2, 8>(ma, mb2, a, tiles512, st, &md)
                  : launch_tc<512, 4, EPI_BIAS, 2, 8>(ma, mb2, a, tiles512, st, &md);
    }
    if (cluster4 == 2 && tma_epi && pad_scratch && row_start == nullptr && per_group > 0 &&
        (N % 8) == 0 && a_gather == nullptr && make_map_out3d(&md, D, G, per_group, N) == 0) {
      // hybrid: the 4-CTA clusters that fit (weight tile multicast across two pairs)
      // plus a 2-CTA instance on the SMs they leave, both pulling two-m-block tiles
      // from one dynamic counter; the instances run on two streams (fork / join)
      CUtensorMap mb4;
      rc = make_map(&mb4, B, b_rows, K, BN / CG / 2);
      if (rc) return rc;
      a.tma_store = 1;
      a.tile_counter = dyn_counter(st, 0, 0, true);
      const int64_t tiles4 = (int64_t)G * ((max_group_rows + 2 * tm - 1) / (2 * tm)) * nblk;
      int nclus = max_clusters4(gelu);
      const int64_t left = num_sms() - 4 * (int64_t)nclus;
      if (a.tile_counter == nullptr || left < 2)
        return gelu ? launch_tc<256, 5, EPI_BIAS_GELU, 2, 8, 4>(ma, mb4, a, tiles4, st, &md)
                    : launch_tc<256, 5, EPI_BIAS, 2, 8, 4>(ma, mb4, a, tiles4, st, &md);
      cudaStream_t side;
      cudaEvent_t fork, join;
      if (!side_stream(&side, &fork, &join)) return MOE_EINVAL;
      cudaEventRecord(fork, st);
      cudaStreamWaitEvent(side, fork, 0);
      int r1 = gelu ? launch_tc<256, 5, EPI_BIAS_GELU, 2, 8, 4>(ma, mb4, a, tiles4, st, &md)
                    : launch_tc<256, 5, EPI_BIAS, 2, 8, 4>(ma, mb4, a, tiles4, st, &md);
      int r2 = gelu ? launch_tc<256, 5, EPI_BIAS_GELU, 2, 8, 2, 2>(ma, mb, a, tiles4, side, &md,
                                                                     left - left % 2)
                    : launch_tc<256, 5, EPI_BIAS, 2, 8, 2, 2>(ma, mb, a, tiles4, side, &md,
                                                             left - left % 2);
      cudaEventRecord(join, side);
      cudaStreamWaitEvent(st, join, 0);
      return r1 ? r1 : r2;
    }
    if (cluster4 == 1 && tma_epi && pad_scratch && row_start == nullptr && per_group > 0 &&
        (N % 8) == 0 && a_gather == nullptr && make_map_out3d(&md, D, G, per_group, N) == 0) {
      // two CTA pairs per cluster (m-blocks 2j, 2j+1) sharing the weight tile by multicast
      CUtensorMap mb4;
      rc = make_map(&mb4, B, b_rows, K, BN / CG / 2);
      if (rc) return rc;
      a.tma_store = 1;
      a.tile_counter = nullptr;  // static schedule: the pairs of a cluster move in step anyway
      const int64_t tiles4 = (int64_t)G * ((max_group_rows + 2 * tm - 1) / (2 * tm)) * nblk;
      return gelu ? launch_tc<256, 5, EPI_BIAS_GELU, 2, 8, 4>(ma, mb4, a, tiles4, st, &md)
                  : launch_tc<256, 5, EPI_BIAS, 2, 8, 4>(ma, mb4, a, tiles4, st, &md);
    }
    if (tma_epi && pad_scratch && row_start == nullptr && per_group > 0 && (N % 8) == 0 &&
        make_map_out3d(&md, D, G, per_group, N) == 0) {
      a.tma_store = 1;
      return gelu ? launch_tc<256, MOE_FWD_STAGES, EPI_BIAS_GELU, 2, MOE_FWD_EW>(ma, mb, a, max_tiles, st, &md)
                  : launch_tc<256, MOE_FWD_STAGES, EPI_BIAS, 2, MOE_FWD_EW>(ma, mb, a, max_tiles, st, &md);
    }
    return gelu ? launch_tc<256, 5, EPI_BIAS_GELU, 2, 8>(ma, mb, a, max_tiles, st)
                : launch_tc<256, 5, EPI_BIAS, 2, 8>(ma, mb, a, max_tiles, st);
  }
#define MOE_TC(BN_, ST_)                                                            \
  return gelu ? launch_tc<BN_, ST_, EPI_BIAS_GELU, 1, (BN_ >= 64 ? 8 : 4)>(ma, mb, a, max_tiles, st) \
              : launch_tc<BN_, ST_, EPI_BIAS, 1, (BN_ >= 64 ? 8 : 4)>(ma, mb, a, max_tiles, st)
  switch (BN) {
    case 32: MOE_TC(32, 8);
    case 64: MOE_TC(64, 8);
    case 128: MOE_TC(128, 6);
    default:
      return gelu ? launch_tc<256, 4, EPI_BIAS_GELU, 1, 4>(ma, mb, a, max_tiles, st)
                  : launch_tc<256, 4, EPI_BIAS, 1, 4>(ma, mb, a, max_tiles, st);
  }
#undef MOE_TC
}

// Residual-MoE layer GEMMs with the shared MLP as extra groups (see EPI_BIAS_RESID):
//   mode 1 (GEMM1): bias + GELU; groups >= a2_group read A rows from A2 (= x)
//   mode 0 (GEMM2): groups < rc_group store y = acc + b2 to D; groups >= rc_group
//                   combine into out (token rows), after every expert tile stored
// Groups are row_stride rows apart (expert buffers: row_stride = capacity; the
// shared groups split the tokens into row_stride-row blocks).
int launch_residual_gemm_bf16(const void* A, int64_t a_rows, const void* A2, int64_t a2_rows,
                              int a2_group, int K, const void* B, int64_t b_rows, int N,
                              const float* bias, void* D, int G, int64_t row_stride,
                              const int32_t* rows, const int32_t* weight_idx,
                              int64_t max_group_rows, int mode, int rc_group, const int32_t* ids,
                              const int32_t* slots, const float* gp, int k, int64_t cap,
                              const void* x, void* out, int64_t S, cudaStream_t st,
                              const int32_t* row_index) {
  if (G < 1 || G > kMaxGroups || K < 8 || (K % 8) || N < 8 || (N % 8) || row_stride < 1)
    return MOE_EINVAL;
  static const int stream_hint = [] {
    const char* v = getenv("MOE_STORE_HINT");
    return v ? atoi(v) : 1;
  }();
  int BN = 256;
  if (N <= 32) BN = 32;
  else if (N <= 64) BN = 64;
  else if (N <= 128) BN = 128;
  const int CG = (BN == 256 && max_group_rows > BM) ? 2 : 1;
  CUtensorMap ma, mb, ma2, md;
  int rc = make_map(&ma, A, a_rows, K, BM);
  if (rc) return rc;
  rc = make_map(&mb, B, b_rows, K, BN / CG);
  if (rc) return rc;
  GemmArgs a{};
  a.bias = bias;
  a.D = (__nv_bfloat16*)D;
  a.K = K;
  a.N = N;
  a.G = G;
  a.row_stride = row_stride;
  a.rows = rows;
  a.weight_idx = weight_idx;
  a.stream_hint = stream_hint;
  const int64_t nblk = (N + BN - 1) / BN;
  const int64_t tm = (int64_t)BM * CG;
  const int64_t max_tiles = (int64_t)G * ((max_group_rows + tm - 1) / tm) * nblk;
  if (max_tiles == 0) return 0;
  if (mode == 1) {
    if (A2 == nullptr || a2_group < 0 || a2_group > G) return MOE_EINVAL;
    rc = make_map(&ma2, A2, a2_rows, K, BM);
    if (rc) return rc;
    a.has_a2 = 1;
    a.a2_group = a2_group;
    a.tile_counter = dyn_counter(st, K, N);
    if (CG == 2) {
      rc = make_map_out3d(&md, D, G, row_stride, N);
      if (rc) return rc;
      a.tma_store = 1;
      return launch_tc<256, MOE_FWD_STAGES, EPI_BIAS_GELU, 2, MOE_FWD_EW>(ma, mb, a, max_tiles, st,
                                                                          &md, 0, &ma2);
    }
    switch (BN) {
      case 32: return launch_tc<32, 8, EPI_BIAS_GELU, 1, 4>(ma, mb, a, max_tiles, st, nullptr, 0, &ma2);
      case 64: return launch_tc<64, 8, EPI_BIAS_GELU, 1, 8>(ma, mb, a, max_tiles, st, nullptr, 0, &ma2);
      case 128: return launch_tc<128, 6, EPI_BIAS_GELU, 1, 8>(ma, mb, a, max_tiles, st, nullptr, 0, &ma2);
      default: return launch_tc<256, 4, EPI_BIAS_GELU, 1, 4>(ma, mb, a, max_tiles, st, nullptr, 0, &ma2);
    }
  }
  if (mode != 0 || rc_group < 0 || rc_group > G || ids == nullptr ||
      (slots == nullptr && row_index == nullptr) || gp == nullptr || x == nullptr ||
      out == nullptr || k < 1 || k > 2)
    return MOE_EINVAL;
  a.c_row_index = row_index;
  a.has_rc = 1;
  a.rc_group = rc_group;
  a.c_ids = ids;
  a.c_slots = slots;
  a.c_gp = gp;
  a.c_k = k;
  a.c_cap = cap;
  a.c_tokens = S;
  a.x_resid = (const __nv_bfloat16*)x;
  a.out = (__nv_bfloat16*)out;
  // the completion counter: a zeroed slot of the per-device pool (graph-safe)
  a.c_done = dyn_counter(st, 0, 0, true);
  if (a.c_done == nullptr) return MOE_EINVAL;
  a.tile_counter = dyn_counter(st, K, N);
  if (CG == 2) {
    if (rc_group > 0) {
      rc = make_map_out3d(&md, D, rc_group, row_stride, N);
      if (rc) return rc;
      a.tma_store = 1;
    }
    // 5 stages: with the 32 KB TMA-store staging, 6 would exceed 227 KB of smem
    return launch_tc<256, 5, EPI_BIAS_RESID, 2, 8>(ma, mb, a, max_tiles, st,
                                                   rc_group > 0 ? &md : nullptr);
  }
  switch (BN) {
    case 32: return launch_tc<32, 8, EPI_BIAS_RESID, 1, 4>(ma, mb, a, max_tiles, st);
    case 64: return launch_tc<64, 8, EPI_BIAS_RESID, 1, 8>(ma, mb, a, max_tiles, st);
    case 128: return launch_tc<128, 6, EPI_BIAS_RESID, 1, 8>(ma, mb, a, max_tiles, st);
    default: return launch_tc<256, 4, EPI_BIAS_RESID, 1, 4>(ma, mb, a, max_tiles, st);
  }
}

// Weight gradients: D = X^T Y per group (see EPI_WGRAD). X: [x_rows, P], Y:
// [x_rows, Q] row-major bf16 (P, Q multiples of 8); K rows of group g start at
// g * k_stride. acc = 0: D bf16 [G, P, Q]; acc = 1: D fp32 [P, Q] += sum over g.
int launch_wgrad_bf16(const void* X, int64_t x_rows, int P, const void* Y, int Q, int G,
                      int64_t k_stride, const int32_t* k_rows, int64_t k_rows_const, void* D,
                      int acc, cudaStream_t st) {
  if (G < 1 || G > kMaxGroups || P < 8 || Q < 8 || (P % 8) || (Q % 8) || x_rows < 0) return MOE_EINVAL;
  static const int stream_hint = [] {
    const char* v = getenv("MOE_STORE_HINT");
    return v ? atoi(v) : 1;
  }();
  const int BN = Q <= 128 ? 128 : 256;
  const int CG = BN == 256 ? 2 : 1;
  CUtensorMap ma, mb;
  // box = 64 columns (one 128-B swizzle line) x 64 token rows
  int rc = make_map(&ma, X, x_rows, P, BK);
  if (rc) return rc;
  rc = make_map(&mb, Y, x_rows, Q, BK);
  if (rc) return rc;
  GemmArgs a{};
  a.N = Q;
  a.K = BK;
  a.G = G;
  a.row_stride = acc ? 0 : P;  // output rows of group g: [g*P, +P) (bf16) or all into [0, P)
  a.rows_const = P;
  a.k_rows = k_rows;
  a.k_rows_const = k_rows_const;
  a.k_stride = k_stride;
  a.D = acc ? nullptr : (__nv_bfloat16*)D;
  a.Dacc = acc ? (float*)D : nullptr;
  a.tile_counter = dyn_counter(st);
  a.stream_hint = acc ? 0 : stream_hint;
  const int64_t tiles = (int64_t)G * ((P + BM * CG - 1) / (BM * CG)) * ((Q + BN - 1) / BN);
  if (x_rows == 0 && acc) return 0;
  if (acc)
    return BN == 256 ? launch_tc<256, 6, EPI_WGRAD_ACC, 2, 8>(ma, mb, a, tiles, st)
                     : launch_tc<128, 6, EPI_WGRAD_ACC, 1, 8>(ma, mb, a, tiles, st);
  CUtensorMap md;
  rc = make_map_out3d(&md, D, G, P, Q);
  if (rc) return rc;
  return BN == 256 ? launch_tc<256, 5, EPI_WGRAD, 2, 8>(ma, mb, a, tiles, st, &md)
                   : launch_tc<128, 5, EPI_WGRAD, 1, 8>(ma, mb, a, tiles, st, &md);
}

int launch_gate_gemm_bf16(const void* x, const void* wg_t, int64_t S, int M, int E, int k,
                          float* logits, int32_t* ids, float* gate_probs, int32_t* local_rank,
                          int32_t* tile_counts, cudaStream_t st, float* probsum) {
  if (S == 0) return 0;
  if (E < 1 || E > 256 || (M % 8) != 0 || k < 1 || k > 2) return MOE_EINVAL;
  int BN = 32;
  while (BN < E) BN *= 2;
  // E >= 128: 2-CTA clusters (M=256 tokens per pair, each CTA loads half of W_g^T per
  // stage) so the smem ring holds more x bytes in flight per SM (the gate is
  // HBM-latency bound: 66 -> ~52 us at C3 measured for the smaller-B configs)
  static const int gate_cg1 = [] {  // MOE_GATE_CG1=1: 1-CTA tiles for E in (64, 128]
    const char* v = getenv("MOE_GATE_CG1");
    return v ? atoi(v) : 0;
  }();
  const int CG = (BN >= 128 && !(gate_cg1 && BN == 128)) ? 2 : 1;
  // MOE_GATE_CL4=1 (E > 64): 4-CTA clusters, two pairs on consecutive 256-token
  // blocks sharing W_g^T by TMA multicast (each CTA loads a quarter per stage).
  // Stand-alone gate 59.4 -> 57.3 us at C3 (L2 flushed) but the layer is 0.4%
  // slower in an interleaved A/B, so pairs stay the default
  static const int cl4_env = [] {
    const char* v = getenv("MOE_GATE_CL4");
    return v ? atoi(v) : 0;
  }();
  const int CLP = (cl4_env == 1 && CG == 2) ? 2 : 1;
  CUtensorMap ma, mb;
  int rc = make_map(&ma, x, S, M, BM);
  if (rc) return rc;
  rc = make_map(&mb, wg_t, BN, M, BN / CG / CLP);  // wg_t is padded to BN rows
  if (rc) return rc;
  GemmArgs a{};
  a.K = M;
  a.N = BN;
  a.G = 1;
  a.row_stride = 0;
  a.rows_const = S;
  a.E = E;
  a.k = k;
  a.S = S;
  a.logits = logits;
  a.ids = ids;
  a.gate_probs = gate_probs;
  a.local_rank = local_rank;
  a.tile_counts = tile_counts;
  a.probsum = probsum;
  a.prefetch = prefetch_mode() & 1 ? 1 : 0;
  // MOE_GATE_BAL=1: per-pair routing-tile ranges balanced to one 128-row routing
  // tile. Parity-green but measured slower (C3 gate 60.4 vs 58.4 us, L2 flushed:
  // profiles/r2_gate_bal.log, with the next-tile L2 prefetch as well:
  // profiles/r2_gate_wave_probe.log) - each SM streams x at a capped rate, so a
  // half pair tile (the leader's 128 rows) takes as long as a full one - so off
  static const int gate_bal = [] {
    const char* v = getenv("MOE_GATE_BAL");
    return v ? atoi(v) : 0;
  }();
  a.gate_bal = (CG == 2 && CLP == 1) ? gate_bal : 0;
  // MOE_GATE_MS=2 (E in (64, 128], pairs): each CTA runs two 128-row sub-tiles against
  // every W_g^T stage (512 tokens per pair tile): the weight crosses L2->SM half as often
  static const int gate_ms = [] {
    const char* v = getenv("MOE_GATE_MS");
    return v ? atoi(v) : 1;
  }();
  if (gate_ms == 2 && CG == 2 && CLP == 1 && BN == 128 && !a.gate_bal) {
    const int64_t tiles2 = (S + 4 * (int64_t)BM - 1) / (4 * (int64_t)BM);
    return launch_tc<128, 5, EPI_GATE, 2, 4, 2, 1, 2>(ma, mb, a, tiles2, st);
  }
  const int64_t tiles = (S + (int64_t)BM * CG * CLP - 1) / ((int64_t)BM * CG * CLP);
  // MOE_GATE_2CTA (default 1; E in (64, 128], pairs): two gate CTAs per SM, each with a
  // 4-stage ring - twice the producer / MMA issue streams per SM. Behind the power-capped
  // GEMM2 (~1 GHz) the gate is issue-bound, not HBM-bound: 80 -> 69 us at base clock,
  // 54 -> 52 us unlocked (profiles/r2_gate_2cta.log)
  static const int gate_2cta = [] {
    const char* v = getenv("MOE_GATE_2CTA");
    return v ? atoi(v) : 1;
  }();
  // (two CTAs per SM only pay when the pair tiles fill more than one CTA per SM;
  // a single-wave launch - decode sizes - keeps the 8-stage ring and prefetches the
  // rest of its tile into L2: 22.8 -> 21.3 us at 64 tokens, cold L2 under ncu)
  const int64_t pairs = num_sms() / (CG * CLP);
  a.prefetch_cur = tiles <= pairs ? 1 : 0;
  if (gate_2cta == 1 && CG == 2 && CLP == 1 && BN == 128 && !a.gate_bal && tiles > pairs)
    return launch_tc<128, 4, EPI_GATE, 2, 4>(ma, mb, a, tiles, st, nullptr, 0, nullptr, 2);
  if (CLP == 2)
    return BN == 128 ? launch_tc<128, 8, EPI_GATE, 2, 4, 4>(ma, mb, a, tiles, st)
                     : launch_tc<256, 6, EPI_GATE, 2, 4, 4>(ma, mb, a, tiles, st);
  switch (BN) {
    case 32: return launch_tc<32, 8, EPI_GATE>(ma, mb, a, tiles, st);
    case 64: return launch_tc<64, 8, EPI_GATE>(ma, mb, a, tiles, st);
    case 128:
      return CG == 1 ? launch_tc<128, 6, EPI_GATE, 1, 4>(ma, mb, a, tiles, st)
                     : launch_tc<128, 8, EPI_GATE, 2, 4>(ma, mb, a, tiles, st);
    default: return launch_tc<256, 6, EPI_GATE, 2, 4>(ma, mb, a, tiles, st);
  }
}

}  // namespace moe

#ifdef MOE_GATE_TRACE
extern "C" int moe_debug_gate_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, moe::g_gate_trace, sizeof(unsigned long long) * 16);
}
#endif
