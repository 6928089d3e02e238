// Grouped expert FFN on tcgen05 / TMEM / TMA (sm_100a).
//
// Replaces the EXPERT_COMPUTE job of the module-based batching schedule
// (reference: pkg/src/moe_planner/offload_dag.py:449-463, cost model hw_profile.py:271-272,288-290)
// with a real kernel.  Numerics follow HF transformers 5.5.0 MixtralExperts.forward
// (modeling_mixtral.py:74-98): gate/up = x @ W_gu^T (bf16 out), h = silu(gate) * up (bf16),
// y = h @ W_d^T (bf16 out).
//
// Layout ("swap-AB", the decode-shaped choice): the weight rows are the MMA M dimension (128 per
// tile) and the routed tokens of one expert are the MMA N dimension (16..256, runtime), so each
// weight tile is streamed from HBM exactly once per token tile while tokens stay L2 resident.
//   gate/up (GATED): the 128-row A tile is 64 gate rows + the 64 matching up rows of W_gu[e]
//            (two 64-row TMA boxes), so TMEM lanes 0-63 hold gate and 64-127 hold up for the same
//            64 features; the epilogue forms bf16(silu(gate)) * up by exchanging the two halves
//            through shared memory.  B = X_perm rows of expert e, K = d.
//   down:    A = 128 rows of W_d[e], B = H rows of expert e, K = f.
// Persistent grid (one CTA per SM), static round-robin over (expert, token-tile, row-tile) units
// ordered row-tile-fastest so concurrently running CTAs share the same token tile in L2.  4-stage
// TMA ring, double-buffered TMEM accumulators (epilogue of unit i overlaps the MMAs of unit i+1).
// Warp roles: w0 = TMA producer, w1 = MMA issuer (+TMEM owner), w2..w5 = epilogue.
#include <cstdlib>

#include "common.cuh"

namespace mgb {

constexpr int kBM = 128;        // weight rows per tile (UMMA M)
constexpr int kBK = 64;         // K per stage (one 128 B swizzle row of bf16)
constexpr int kBNMax = 256;     // max tokens per tile (UMMA N)
constexpr int kBRows = 32;      // token rows per TMA box
constexpr int kATileBytes = kBM * kBK * 2;         // 16 KB
constexpr int kAHalfBytes = kATileBytes / 2;       // 8 KB (64 rows)
constexpr int kBTileBytes = kBNMax * kBK * 2;      // 32 KB
constexpr int kBBoxBytes = kBRows * kBK * 2;       // 4 KB
constexpr int kMaxExperts = 256;
constexpr int kStages = 4;
constexpr int kStageBytes = kATileBytes + kBTileBytes;
constexpr int kAccStages = 2;                      // 2 x 256 TMEM columns
constexpr int kXStride = 33;                       // padded row of the gate/up exchange buffer
// epilogue warp groups (4 warps each, one per TMEM lane quarter): the gated epilogue (SiLU*up with a
// shared-memory exchange) is the critical path of the gate/up GEMM at DeepSeek shapes, so it gets two
// groups working on alternate 32-token chunks; the plain epilogue keeps one
#ifndef MGB_GATED_EPI_GROUPS
#define MGB_GATED_EPI_GROUPS 2
#endif
template <bool GATED> struct Epi {
  static constexpr int kGroups = GATED ? MGB_GATED_EPI_GROUPS : 1;
  static constexpr int kThreads = 64 + kGroups * 128;  // TMA warp + MMA warp + epilogue warps
  static constexpr int kXBytes = GATED ? kGroups * 64 * kXStride * 4 : 0;  // gate/up exchange buffers
};
template <bool GATED> constexpr int gemm_smem() {
  return kStages * kStageBytes + Epi<GATED>::kXBytes + 1024 /*align*/ + 256 /*barriers*/;
}

// Token tiles of an expert: as few as fit N <= 256.  The gated GEMM (heavier per-token epilogue)
// sizes them equally (multiple of 32) so no unit is a tiny remainder whose epilogue cannot hide
// behind the next unit's main loop (568 tokens -> 3 x 192 rather than 256 + 256 + 56); the plain
// GEMM keeps full 256-token tiles, which measured faster for it.
MGB_DEVINL int token_tile(int cnt, bool balanced) {
  if (!balanced) return kBNMax;
  const int nt0 = (cnt + kBNMax - 1) / kBNMax;
  return nt0 == 0 ? kBNMax : (((cnt + nt0 - 1) / nt0) + 31) & ~31;
}
MGB_DEVINL int token_tiles(int cnt, bool balanced) {
  const int t = token_tile(cnt, balanced);
  return (cnt + t - 1) / t;
}

struct UnitSched {
  const int* s_prefix;  // [E+1] units before expert e (smem)
  int E, MT;
  bool balanced;
  __device__ void decode(int u, const int* offs, int& e, int& nt, int& mt, int& tok0, int& n) const {
    int lo = 0, hi = E - 1;  // last e with prefix[e] <= u
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s_prefix[mid] <= u) lo = mid; else hi = mid - 1;
    }
    e = lo;
    int local = u - s_prefix[e];
    const int beg = offs[e], cnt = offs[e + 1] - beg;
    // token tiles fastest: the (up to ceil(cnt/256)) units that share one weight tile run on
    // neighbouring CTAs at the same time, so the tile is read from HBM once and hit in L2 after
    const int tile = token_tile(cnt, balanced), NT = (cnt + tile - 1) / tile;
    mt = local / NT;
    nt = local - mt * NT;
    tok0 = beg + nt * tile;
    n = min(tile, cnt - nt * tile);
  }
};

// Wait-time accounting of the fused FFN kernel (build with -DMGB_GEMM_TRACE; tools/ffn_trace.py):
// g_ffn_trace[cta][i] = cycles spent in: 0 producer empty waits, 1 MMA full waits, 2 MMA TMEM-empty
// waits, 3 epilogue TMEM-full waits (warp 2), 4 producer dependency waits, 5 kernel cycles (thread 0)
#ifdef MGB_GEMM_TRACE
__device__ long long g_ffn_trace[256][8];
#define FFN_T0() const long long _t0 = clock64()
#define FFN_ACC(i) g_ffn_trace[blockIdx.x][i] += clock64() - _t0
#else
#define FFN_T0()
#define FFN_ACC(i)
#endif

MGB_DEVINL int ld_acquire_gpu_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// named barrier of one epilogue group (ids 1.., 128 threads); 0 is __syncthreads
MGB_DEVINL void epi_bar(int group) { asm volatile("bar.sync %0, 128;" ::"r"(1 + group) : "memory"); }

// One 32-token chunk of the gated epilogue.  TMEM lanes 0-63 hold gate, 64-127 up for the same 64
// features; the gate warps finish tokens 0-15 of the chunk and the up warps tokens 16-31, each
// taking the partner half through shared memory, so all four epilogue warps do the SiLU*up work.
// h = bf16(bf16(silu(bf16(gate))) * bf16(up)) (HF MixtralExperts, modeling_mixtral.py:91-93).
MGB_DEVINL void gated_chunk(uint32_t tl, int c0, int n, bool is_up, int f, float* xbuf, __nv_bfloat16* ocol,
                            int ldo, int group) {
  uint32_t v[32];
  tmem_ld32(tl + c0, v);
  tmem_ld_wait();
  float* xr = xbuf + f * kXStride;
  if (is_up) {  // hand over up for tokens 0-15, finish tokens 16-31 (register indices stay static)
#pragma unroll
    for (int j = 0; j < 16; ++j) xr[j] = bf16_round(__uint_as_float(v[j]));
  } else {      // hand over gate for tokens 16-31, finish tokens 0-15
#pragma unroll
    for (int j = 0; j < 16; ++j) xr[16 + j] = bf16_round(__uint_as_float(v[16 + j]));
  }
  epi_bar(group);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int c = c0 + (is_up ? 16 : 0) + j;
    const float mine = bf16_round(__uint_as_float(is_up ? v[16 + j] : v[j]));
    const float other = is_up ? xr[16 + j] : xr[j];
    const float gv = is_up ? other : mine, uv = is_up ? mine : other;
    // silu in fp32 with the SFU exponential and a fast divide (within bf16 rounding of HF's silu)
    if (c < n) ocol[(size_t)c * ldo] = __float2bfloat16_rn(bf16_round(__fdividef(gv, 1.0f + __expf(-gv))) * uv);
  }
  epi_bar(group);
}

template <bool GATED, bool ROWPTR = false>
__global__ void __launch_bounds__(Epi<GATED>::kThreads, 1)
moe_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const int* __restrict__ offsets, int E, int MT, int K, int rows_per_expert, int half_rows,
                __nv_bfloat16* __restrict__ out, int ldo, bool balanced,
                const long long* __restrict__ row_ptr, int rows_cap, int* __restrict__ cap_status) {
  mgb::pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tiles = smem;
  float* xbuf = reinterpret_cast<float*>(smem + kStages * kStageBytes);  // [group][64][kXStride] exchange
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes + Epi<GATED>::kXBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + kAccStages);
  __shared__ int s_prefix[kMaxExperts + 1];

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  constexpr int kRowsPerUnit = GATED ? kBM / 2 : kBM;  // output features per unit

  // unit prefix over experts: units(e) = ceil(n_e / BN) * MT
  if (threadIdx.x == 0) {
    int acc = 0;
    const bool fit = segments_fit(offsets, E, rows_cap, cap_status, GATED ? kCapGateUp : kCapDown);
    for (int e = 0; e < E; ++e) {
      s_prefix[e] = acc;
      const int cnt = offsets[e + 1] - offsets[e];
      acc += token_tiles(cnt, balanced) * MT;
    }
    s_prefix[E] = fit ? acc : 0;  // overflow: no unit runs (status recorded), nothing is written
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < kAccStages; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], Epi<GATED>::kGroups * 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = s_prefix[E];
  UnitSched sched{s_prefix, E, MT, balanced};
  const int KB = K / kBK;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int e, nt, mt, tok0, n;
        sched.decode(u, offsets, e, nt, mt, tok0, n);
        const int nb = (n + kBRows - 1) / kBRows;
        const uint32_t bytes = kATileBytes + nb * kBBoxBytes;
        const int arow0 = e * rows_per_expert + mt * kRowsPerUnit;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], bytes);
          uint8_t* st = tiles + stage * kStageBytes;
          if (GATED) {
            tma_load_2d(st, &tmA, &full_bar[stage], kb * kBK, arow0, pol_w);                          // gate
            tma_load_2d(st + kAHalfBytes, &tmA, &full_bar[stage], kb * kBK, arow0 + half_rows, pol_w);  // up
          } else {
            tma_load_2d(st, &tmA, &full_bar[stage], kb * kBK, arow0, pol_w);
          }
          uint8_t* bt = st + kATileBytes;
          for (int j = 0; j < nb; ++j)
            tma_load_2d(bt + j * kBBoxBytes, &tmB, &full_bar[stage], kb * kBK, tok0 + j * kBRows, pol_x);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int e, nt, mt, tok0, n;
        sched.decode(u, offsets, e, nt, mt, tok0, n);
        const uint32_t N = (uint32_t)((n + 15) & ~15);
        const uint32_t idesc = make_idesc_bf16(kBM, N);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * kBNMax;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(tiles + stage * kStageBytes);
          const uint64_t a0 = make_sdesc_sw128(st);
          const uint64_t b0 = make_sdesc_sw128(st + kATileBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)  // +32 B per 16-element K step (desc units of 16 B)
            umma_bf16(d0, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) ? 1u : 0u);
          umma_commit(&empty_bar[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull_bar[acc]);
        if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------ epilogue (warps 2..5) ------------------------------
    const uint32_t q = warp & 3;          // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;        // accumulator row (lane) of this thread
    const int group = Epi<GATED>::kGroups > 1 ? (int)(warp - 2) >> 2 : 0;  // column group (32-token chunks)
    float* gx = xbuf + group * 64 * kXStride;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      int e, nt, mt, tok0, n;
      sched.decode(u, offsets, e, nt, mt, tok0, n);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tl = tmem_base + ((q * 32) << 16) + acc * kBNMax;
      if (GATED) {
        // quarters 0,1: gate rows 0..63; quarters 2,3: up rows 0..63 (same features)
        const bool is_up = q >= 2;
        const int f = row & 63;
        __nv_bfloat16* ocol = out + (size_t)tok0 * ldo + mt * kRowsPerUnit + f;
        for (int c0 = 32 * group; c0 < n; c0 += 32 * Epi<GATED>::kGroups) gated_chunk(tl, c0, n, is_up, f, gx, ocol, ldo, group);
      } else {
        const int col = mt * kRowsPerUnit + row;
        __nv_bfloat16* ocol = out + (size_t)tok0 * ldo + col;
        for (int c0 = 32 * group; c0 < n; c0 += 32 * Epi<GATED>::kGroups) {
          uint32_t v[32];
          tmem_ld32(tl + c0, v);
          tmem_ld_wait();
          if (ROWPTR) {  // row stores to per-row destinations (EP combine, layout transposes)
            // one coalesced load of the chunk's 32 row pointers, broadcast lane by lane
            const long long mine = c0 + (int)lane < n ? row_ptr[tok0 + c0 + lane] : 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const long long p = __shfl_sync(0xffffffffu, mine, j);
              if (p) reinterpret_cast<__nv_bfloat16*>(p)[col] = __float2bfloat16_rn(__uint_as_float(v[j]));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < n) ocol[(size_t)(c0 + j) * ldo] = __float2bfloat16_rn(__uint_as_float(v[j]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem_base);
}

// ------------------------------------------------------------------------------------------
// CTA-pair variant (cluster of 2, tcgen05 cta_group::2, UMMA M = 256).  Each CTA holds its own
// 128 weight rows (A) and HALF of the token tile (B rows), so per SM the token-operand smem and
// L2 traffic halve and the ring deepens to 6 stages; the leader CTA issues the pair MMAs and
// multicasts its commits to both CTAs' barriers; both CTAs' TMA loads complete on the leader's
// full barrier; both epilogues drain their own TMEM half and arrive on the leader's TMEM-empty
// barrier.  Unit = (expert, token tile, 256-row pair tile).
// ------------------------------------------------------------------------------------------
constexpr int kPStages = 6;
// A CTA's half of the token tile (N/2 rows, a multiple of 8) is loaded as boxes of 64 / 32 / 16 / 8
// rows (N = 208: 64 + 32 + 8 -- three TMA requests instead of seven 16-row ones).  The TMA request
// count, not the bytes, is what bounded the ring: streaming Mixtral's W_gate_up at 64-row A boxes with
// a 104-row B slice per stage runs at 4.1 TB/s of A with 16-row B boxes and at 6.5 TB/s -- the A-only
// rate -- with 64+32+8 (tools/tma_pattern_bench.cu).  Every box starts on a whole 8-row (1 KB) swizzle
// atom, so the boxes together land exactly where one tall box would.
// With one map per box height 8, 16, ..., 128 rows the half tile is ONE request (`one`, MGB_TMA1 on by
// default): gate/up stages then take 2 requests (one 4-D gate+up A box, one B box) instead of 5, down
// stages 2 instead of 4 -- Mixtral's fused FFN 17.47 -> 16.68 ms per replayed forward (same box).
constexpr int kBMaps = kBNMax / 2 / 8;  // box heights 8 * (i + 1) rows
struct BMaps {
  CUtensorMap m[kBMaps];  // box width kBK
};
MGB_DEVINL void load_b_rows_pair(uint8_t* bt, const BMaps& mp, uint64_t* bar, int kcol, int row0, int rows,
                                 uint64_t pol, bool one = false) {
  if (one) {
    tma_load_2d_pair(bt, &mp.m[rows / 8 - 1], bar, kcol, row0, pol);
    return;
  }
  int r = 0;
  for (; rows - r >= 64; r += 64) tma_load_2d_pair(bt + r * 128, &mp.m[7], bar, kcol, row0 + r, pol);
  if (rows - r >= 32) { tma_load_2d_pair(bt + r * 128, &mp.m[3], bar, kcol, row0 + r, pol); r += 32; }
  if (rows - r >= 16) { tma_load_2d_pair(bt + r * 128, &mp.m[1], bar, kcol, row0 + r, pol); r += 16; }
  if (rows - r >= 8) tma_load_2d_pair(bt + r * 128, &mp.m[0], bar, kcol, row0 + r, pol);
}
MGB_DEVINL void prefetch_bmaps(const BMaps& mp) {
#pragma unroll
  for (int i = 0; i < kBMaps; ++i) prefetch_tmap(&mp.m[i]);
}
constexpr int kPStageBytes = kATileBytes + (kBNMax / 2) * kBK * 2;  // 16 KB A + <= 16 KB half-B
template <bool GATED> constexpr int pair_smem() {
  return kPStages * kPStageBytes + Epi<GATED>::kXBytes + 1024 + 256;
}

template <bool GATED, bool ROWPTR = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Epi<GATED>::kThreads, 1)
moe_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ BMaps tmB,
                     const __grid_constant__ CUtensorMap tmA4,  // GATED: W as [E][gate|up][f][K] (one box per stage)
                     const int* __restrict__ offsets, int E, int MT, int K, int rows_per_expert, int half_rows,
                     __nv_bfloat16* __restrict__ out, int ldo, bool balanced,
                     const long long* __restrict__ row_ptr, int nalign, int rows_cap, int* __restrict__ cap_status,
                     int tma1) {
  mgb::pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tiles = smem;
  float* xbuf = reinterpret_cast<float*>(smem + kPStages * kPStageBytes);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kPStages * kPStageBytes + Epi<GATED>::kXBytes);
  uint64_t* empty_bar = full_bar + kPStages;
  uint64_t* tfull_bar = empty_bar + kPStages;
  uint64_t* tempty_bar = tfull_bar + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + kAccStages);
  __shared__ int s_prefix[kMaxExperts + 1];

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  constexpr int kRowsPerCta = GATED ? kBM / 2 : kBM;  // output features per CTA per unit

  if (threadIdx.x == 0) {
    int acc = 0;
    const bool fit = segments_fit(offsets, E, rows_cap, cap_status, GATED ? kCapGateUp : kCapDown);
    for (int e = 0; e < E; ++e) {
      s_prefix[e] = acc;
      const int cnt = offsets[e + 1] - offsets[e];
      acc += token_tiles(cnt, balanced) * MT;
    }
    s_prefix[E] = fit ? acc : 0;  // overflow: no unit runs (status recorded), nothing is written
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(GATED && tma1 ? &tmA4 : &tmA);
    prefetch_bmaps(tmB);
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < kAccStages; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * 4 * Epi<GATED>::kGroups);  // both CTAs' epilogue warps (used on the leader)
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = s_prefix[E];
  UnitSched sched{s_prefix, E, MT, balanced};
  const int KB = K / kBK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
#ifdef MGB_GEMM_TRACE
  const long long _kt0 = clock64();
#endif

  if (warp == 0) {
    // ------------------------------ TMA producer (both CTAs) ------------------------------
    if (elect_one()) {
      // a weight tile read by several token tiles (neighbouring pairs, same time) stays in L2 for
      // them; one read once streams past it
      const uint64_t pol_once = policy_evict_first(), pol_shared = policy_evict_normal();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < total; u += npairs) {
        int e, nt, mt, tok0, n;
        sched.decode(u, offsets, e, nt, mt, tok0, n);
        const uint64_t pol_w = token_tiles(offsets[e + 1] - offsets[e], balanced) > 1 ? pol_shared : pol_once;
        const int N = (n + nalign - 1) & ~(nalign - 1);
        const int half = N / 2;
        const uint32_t bytes = 2u * (kATileBytes + half * kBK * 2);
        const int arow0 = e * rows_per_expert + mt * 2 * kRowsPerCta + rank * kRowsPerCta;
        const int trow0 = tok0 + rank * half;
        for (int kb = 0; kb < KB; ++kb) {
          { FFN_T0(); mbar_wait(&empty_bar[stage], phase ^ 1); FFN_ACC(0); }
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], bytes);
          uint8_t* st = tiles + stage * kPStageBytes;
          if (GATED && tma1) {
            tma_load_4d_pair(st, &tmA4, &full_bar[stage], kb * kBK, arow0 - e * rows_per_expert, 0, e, pol_w);
          } else if (GATED) {
            tma_load_2d_pair(st, &tmA, &full_bar[stage], kb * kBK, arow0, pol_w);
            tma_load_2d_pair(st + kAHalfBytes, &tmA, &full_bar[stage], kb * kBK, arow0 + half_rows, pol_w);
          } else {
            tma_load_2d_pair(st, &tmA, &full_bar[stage], kb * kBK, arow0, pol_w);
          }
          load_b_rows_pair(st + kATileBytes, tmB, &full_bar[stage], kb * kBK, trow0, half, pol_x, tma1 != 0);
          if (++stage == kPStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (leader only) ------------------------------
    if (leader && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < total; u += npairs) {
        int e, nt, mt, tok0, n;
        sched.decode(u, offsets, e, nt, mt, tok0, n);
        const uint32_t N = (uint32_t)((n + nalign - 1) & ~(nalign - 1));
        const uint32_t idesc = make_idesc_bf16(2 * kBM, N);
        { FFN_T0(); mbar_wait(&tempty_bar[acc], acc_phase ^ 1); FFN_ACC(2); }
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * kBNMax;
        for (int kb = 0; kb < KB; ++kb) {
          { FFN_T0(); mbar_wait(&full_bar[stage], phase); FFN_ACC(1); }
          tc_fence_after();
          const uint32_t st = smem_u32(tiles + stage * kPStageBytes);
          const uint64_t a0 = make_sdesc_sw128(st);
          const uint64_t b0 = make_sdesc_sw128(st + kATileBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16_pair(d0, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) ? 1u : 0u);
          umma_commit_pair(&empty_bar[stage], 0x3);
          if (++stage == kPStages) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&tfull_bar[acc], 0x3);
        if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------ epilogue (warps 2..5, both CTAs) ------------------------------
    const uint32_t q = warp & 3;
    const int row = q * 32 + lane;
    const int group = Epi<GATED>::kGroups > 1 ? (int)(warp - 2) >> 2 : 0;
    float* gx = xbuf + group * 64 * kXStride;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < total; u += npairs) {
      int e, nt, mt, tok0, n;
      sched.decode(u, offsets, e, nt, mt, tok0, n);
      if (warp == 2 && lane == 0) { FFN_T0(); mbar_wait(&tfull_bar[acc], acc_phase); FFN_ACC(3); }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tl = tmem_base + ((q * 32) << 16) + acc * kBNMax;
      const int col0 = mt * 2 * kRowsPerCta + rank * kRowsPerCta;
      if (GATED) {
        const bool is_up = q >= 2;
        const int f = row & 63;
        __nv_bfloat16* ocol = out + (size_t)tok0 * ldo + col0 + f;
        for (int c0 = 32 * group; c0 < n; c0 += 32 * Epi<GATED>::kGroups) gated_chunk(tl, c0, n, is_up, f, gx, ocol, ldo, group);
      } else {
        const int col = col0 + row;
        __nv_bfloat16* ocol = out + (size_t)tok0 * ldo + col;
        for (int c0 = 32 * group; c0 < n; c0 += 32 * Epi<GATED>::kGroups) {
          uint32_t v[32];
          tmem_ld32(tl + c0, v);
          tmem_ld_wait();
          if (ROWPTR) {  // row stores to per-row destinations (EP combine, layout transposes)
            // one coalesced load of the chunk's 32 row pointers, broadcast lane by lane
            const long long mine = c0 + (int)lane < n ? row_ptr[tok0 + c0 + lane] : 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const long long p = __shfl_sync(0xffffffffu, mine, j);
              if (p) reinterpret_cast<__nv_bfloat16*>(p)[col] = __float2bfloat16_rn(__uint_as_float(v[j]));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c0 + j < n) ocol[(size_t)(c0 + j) * ldo] = __float2bfloat16_rn(__uint_as_float(v[j]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
      if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_pair<512>(tmem_base);
#ifdef MGB_GEMM_TRACE
  if (threadIdx.x == 0) g_ffn_trace[blockIdx.x][5] = clock64() - _kt0;
#endif
}

// ------------------------------------------------------------------------------------------
// Fused expert FFN: gate/up AND down of every expert in ONE persistent CTA-pair launch.
// The unit list is [all gate/up units | all down units] (each part ordered as the separate kernels
// order theirs); pair p runs units p, p + npairs, ... .  A down unit of expert e needs all of e's
// h rows: its producers wait until the epilogue warps of every gate/up unit of e have stored their
// rows and counted them on done[e] (release: fence + atomic; acquire + proxy fence before the TMA
// reads h).  No deadlock: a pair reaches a down unit only after issuing all of its own gate/up
// units, every gate/up unit precedes every down unit in the list, and the persistent grid is
// co-resident.  What it buys: the two launches' wave tails (Mixtral: 896 gate/up units of 64 K
// blocks then 128 down units of 224 on 74 pairs: 13 + 2 rounds) become one tail, and the gap
// between the launches disappears.  The last pair to finish zeroes done[] for the next launch.
// ------------------------------------------------------------------------------------------
struct FfnGemm {
  int MT;               // pair row tiles per expert
  int KB;               // K blocks
  int rows_per_expert;  // weight rows per expert (2f gated, d down)
  int half_rows;        // f (gated: offset of the up rows)
  int ldo;              // output row stride
  __nv_bfloat16* out;
};

MGB_DEVINL void ffn_decode(int u, int total_gu, const int* s_pgu, const int* s_pdn, int E, const int* offs,
                           const FfnGemm& gu, const FfnGemm& dn, bool& gated, int& e, int& mt, int& tok0, int& n) {
  gated = u < total_gu;
  const int* pre = gated ? s_pgu : s_pdn;
  const int v = gated ? u : u - total_gu;
  int lo = 0, hi = E - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= v) lo = mid; else hi = mid - 1;
  }
  e = lo;
  const int local = v - pre[e];
  const int beg = offs[e], cnt = offs[e + 1] - beg;
  const int tile = token_tile(cnt, gated), NT = (cnt + tile - 1) / tile;
  mt = local / NT;
  const int nt = local - mt * NT;
  tok0 = beg + nt * tile;
  n = min(tile, cnt - nt * tile);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Epi<true>::kThreads, 1)
moe_ffn_pair_kernel(const __grid_constant__ CUtensorMap tmAg,  // W_gate_up [E][gate|up][f][K/64][64], 5-D
                    const __grid_constant__ BMaps tmBx,        // x_perm [rows][K/64][64], 3-D
                    const __grid_constant__ CUtensorMap tmAd,  // W_down [E*d][f/64][64], 3-D
                    const __grid_constant__ BMaps tmBh,        // h [rows][f/64][64], 3-D
                    const int* __restrict__ offsets, int E, FfnGemm gu, FfnGemm dn, int nalign, int rows_cap,
                    int* __restrict__ cap_status, int* __restrict__ done, int kps) {
  mgb::pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tiles = smem;
  float* xbuf = reinterpret_cast<float*>(smem + kPStages * kPStageBytes);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kPStages * kPStageBytes + Epi<true>::kXBytes);
  uint64_t* empty_bar = full_bar + kPStages;
  uint64_t* tfull_bar = empty_bar + kPStages;
  uint64_t* tempty_bar = tfull_bar + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + kAccStages);
  __shared__ int s_pgu[kMaxExperts + 1], s_pdn[kMaxExperts + 1], s_need[kMaxExperts];
  __shared__ bool s_last;
  constexpr int kGroups = Epi<true>::kGroups;
  constexpr int kArrivals = 2 * 4 * kGroups;  // epilogue warps of both CTAs per unit

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int nst = kPStages / kps;  // ring stages of kps K-blocks each

  if (threadIdx.x == 0) {
    const bool fit = segments_fit(offsets, E, rows_cap, cap_status, kCapGateUp);
    int ag = 0, ad = 0;
    for (int e = 0; e < E; ++e) {
      s_pgu[e] = ag;
      s_pdn[e] = ad;
      const int cnt = offsets[e + 1] - offsets[e];
      const int ug = token_tiles(cnt, true) * gu.MT;
      s_need[e] = ug * kArrivals;
      ag += ug;
      ad += token_tiles(cnt, false) * dn.MT;
    }
    s_pgu[E] = fit ? ag : 0;
    s_pdn[E] = fit ? ad : 0;
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmAg);
    prefetch_bmaps(tmBx);
    prefetch_tmap(&tmAd);
    prefetch_bmaps(tmBh);
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < kAccStages; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], kArrivals);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_gu = s_pgu[E];
  const int total = total_gu + s_pdn[E];
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
#ifdef MGB_GEMM_TRACE
  const long long _kt0 = clock64();
#endif

  if (warp == 0) {
    // ------------------------------ TMA producer (both CTAs) ------------------------------
    if (elect_one()) {
      const uint64_t pol_once = policy_evict_first(), pol_shared = policy_evict_normal();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < total; u += npairs) {
        bool gated;
        int e, mt, tok0, n;
        ffn_decode(u, total_gu, s_pgu, s_pdn, E, offsets, gu, dn, gated, e, mt, tok0, n);
        const FfnGemm& G = gated ? gu : dn;
        const BMaps& tB = gated ? tmBx : tmBh;
        if (!gated) {  // h rows of expert e: every gate/up unit of e has stored and counted them
          const int need = s_need[e];
          {
            FFN_T0();
            while (ld_acquire_gpu_s32(done + e) < need) __nanosleep(64);
            FFN_ACC(4);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        const int rows_cta = gated ? kBM / 2 : kBM;
        const uint64_t pol_w = token_tiles(offsets[e + 1] - offsets[e], gated) > 1 ? pol_shared : pol_once;
        const int N = (n + nalign - 1) & ~(nalign - 1);
        const int half = N / 2;
        const uint32_t bytes = 2u * kps * (kATileBytes + half * kBK * 2);
        const int arow0 = e * G.rows_per_expert + mt * 2 * rows_cta + rank * rows_cta;
        const int trow0 = tok0 + rank * half;
        const CUtensorMap* tBm = &tB.m[half / 8 - 1];
        // one stage = kps K-blocks: [A kb0 | A kb1 | B kb0 | B kb1], ONE request per operand
        for (int kb = 0; kb < G.KB; kb += kps) {
          { FFN_T0(); mbar_wait(&empty_bar[stage], phase ^ 1); FFN_ACC(0); }
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], bytes);
          uint8_t* st = tiles + stage * kps * kPStageBytes;
          if (gated)  // gate rows then the matching up rows of every K-block
            tma_load_5d_pair(st, &tmAg, &full_bar[stage], 0, (mt * 2 + (int)rank) * rows_cta, 0, e, kb, pol_w);
          else
            tma_load_3d_pair(st, &tmAd, &full_bar[stage], 0, arow0, kb, pol_w);
          tma_load_3d_pair(st + kps * kATileBytes, tBm, &full_bar[stage], 0, trow0, kb, pol_x);
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (leader only) ------------------------------
    if (leader && elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = pair; u < total; u += npairs) {
        bool gated;
        int e, mt, tok0, n;
        ffn_decode(u, total_gu, s_pgu, s_pdn, E, offsets, gu, dn, gated, e, mt, tok0, n);
        const int KB = gated ? gu.KB : dn.KB;
        const uint32_t N = (uint32_t)((n + nalign - 1) & ~(nalign - 1));
        const uint32_t idesc = make_idesc_bf16(2 * kBM, N);
        { FFN_T0(); mbar_wait(&tempty_bar[acc], acc_phase ^ 1); FFN_ACC(2); }
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * kBNMax;
        const uint32_t bstride = (N / 2) * kBK * 2;  // B bytes of one K-block (this CTA's half)
        for (int kb = 0; kb < KB; kb += kps) {
          { FFN_T0(); mbar_wait(&full_bar[stage], phase); FFN_ACC(1); }
          tc_fence_after();
          const uint32_t st = smem_u32(tiles + stage * kps * kPStageBytes);
          for (int j = 0; j < kps; ++j) {
            const uint64_t a0 = make_sdesc_sw128(st + j * kATileBytes);
            const uint64_t b0 = make_sdesc_sw128(st + kps * kATileBytes + j * bstride);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16_pair(d0, a0 + 2 * k, b0 + 2 * k, idesc, ((kb + j) | k) ? 1u : 0u);
          }
          umma_commit_pair(&empty_bar[stage], 0x3);
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&tfull_bar[acc], 0x3);
        if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------ epilogue (warps 2..9, both CTAs) ------------------------------
    const uint32_t q = warp & 3;
    const int row = q * 32 + lane;
    const int group = (int)(warp - 2) >> 2;
    float* gx = xbuf + group * 64 * kXStride;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = pair; u < total; u += npairs) {
      bool gated;
      int e, mt, tok0, n;
      ffn_decode(u, total_gu, s_pgu, s_pdn, E, offsets, gu, dn, gated, e, mt, tok0, n);
      if (warp == 2 && lane == 0) { FFN_T0(); mbar_wait(&tfull_bar[acc], acc_phase); FFN_ACC(3); }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tl = tmem_base + ((q * 32) << 16) + acc * kBNMax;
      if (gated) {
        const int col0 = mt * 2 * (kBM / 2) + rank * (kBM / 2);
        const bool is_up = q >= 2;
        const int f = row & 63;
        __nv_bfloat16* ocol = gu.out + (size_t)tok0 * gu.ldo + col0 + f;
        for (int c0 = 32 * group; c0 < n; c0 += 32 * kGroups) gated_chunk(tl, c0, n, is_up, f, gx, ocol, gu.ldo, group);
      } else {
        const int col = mt * 2 * kBM + rank * kBM + row;
        __nv_bfloat16* ocol = dn.out + (size_t)tok0 * dn.ldo + col;
        for (int c0 = 32 * group; c0 < n; c0 += 32 * kGroups) {
          uint32_t v[32];
          tmem_ld32(tl + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < n) ocol[(size_t)(c0 + j) * dn.ldo] = __float2bfloat16_rn(__uint_as_float(v[j]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (gated) {  // this warp's share of e's h rows is stored: count it (release to the down units)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(done + e, 1);
      }
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
      if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc_pair<512>(tmem_base);
#ifdef MGB_GEMM_TRACE
  if (threadIdx.x == 0) g_ffn_trace[blockIdx.x][5] = clock64() - _kt0;
#endif
  // the last CTA out resets the per-expert counters (and the exit ticket) for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done + kMaxExperts, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) done[e] = 0;
    if (threadIdx.x == 0) done[kMaxExperts] = 0;
  }
}

}  // namespace mgb

// ------------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------------
namespace {
// one TMA request per operand per stage in the pair kernels (4-D gate+up A box, exact-height B box);
// MGB_TMA1=0 restores the 2 + (up to 4) request split
int tma1_enabled() {
  static const int v = [] {
    const char* e = getenv("MGB_TMA1");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}

// [E][2][f][K] view of a gated weight [E, 2f, K]: one box = 64 gate rows + the matching 64 up rows
int encode_gate_up_4d(CUtensorMap* m, const void* w, int E, int f, int K) {
  const uint64_t dims[4] = {(uint64_t)K, (uint64_t)f, 2, (uint64_t)E};
  const uint64_t strides[3] = {(uint64_t)K * 2, (uint64_t)f * K * 2, (uint64_t)2 * f * K * 2};
  const uint32_t box[4] = {(uint32_t)mgb::kBK, (uint32_t)mgb::kBM / 2, 2, 1};
  return mgb_host::encode_tmap_bf16(m, w, 4, dims, strides, box, true, true) != CUDA_SUCCESS;
}

bool use_pair_kernel() {
  static const bool v = [] {
    const char* e = getenv("MGB_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return v;
}

// token-operand maps of the pair kernels: box heights 64 / 32 / 16 / 8 rows over [rows, K] bf16
int encode_bmaps(mgb::BMaps* mp, const void* act, int K, int rows) {
  for (int i = 0; i < mgb::kBMaps; ++i)
    if (mgb_host::encode_tmap_2d_bf16(&mp->m[i], act, K, rows, (uint64_t)K * 2, mgb::kBK, 8 * (i + 1)) != CUDA_SUCCESS)
      return 1;
  return 0;
}

// K-blocked token maps of the fused FFN kernel: [rows][K/64][64] with boxes of 8 * (i + 1) rows x kps
// K-blocks (smem image: kps consecutive [rows][64] swizzled tiles)
int encode_bmaps_kb(mgb::BMaps* mp, const void* act, int K, int rows, int kps) {
  const uint64_t dims[3] = {(uint64_t)mgb::kBK, (uint64_t)rows, (uint64_t)K / mgb::kBK};
  const uint64_t strides[2] = {(uint64_t)K * 2, (uint64_t)mgb::kBK * 2};
  for (int i = 0; i < mgb::kBMaps; ++i) {
    const uint32_t box[3] = {(uint32_t)mgb::kBK, (uint32_t)(8 * (i + 1)), (uint32_t)kps};
    if (mgb_host::encode_tmap_bf16(&mp->m[i], act, 3, dims, strides, box, true, true) != CUDA_SUCCESS) return 1;
  }
  return 0;
}

template <bool GATED, bool PAIR, bool ROWPTR>
int launch_variant(const CUtensorMap& tmA, const CUtensorMap& tmA4, const CUtensorMap& tmB, const mgb::BMaps& tmBs,
                   const int* offsets, int E, int MT, int K,
                   int rows_per_expert, int half_rows, void* out, int ldo, bool balanced, const long long* row_ptr,
                   int rows_cap, cudaStream_t stream) {
  int* cap_status = mgb_host::capacity_status_ptr();
  if (!cap_status) return MGB_ECUDA;
  if (PAIR) {
    if (const int rc = mgb_host::ensure_max_smem((const void*)mgb::moe_gemm_pair_kernel<GATED, ROWPTR>,
                                                 mgb::pair_smem<GATED>()))
      return rc;
    const int grid = mgb_host::num_sms() & ~1;
    // pair MMA N: a multiple of 16 (each CTA holds N/2 token rows, whole 8-row swizzle atoms);
    // MGB_PAIR_NALIGN=32 pads further
    static const int nalign = [] {
      const char* e = getenv("MGB_PAIR_NALIGN");
      return (e && atoi(e) == 32) ? 32 : 16;
    }();
    mgb_host::launch(mgb::moe_gemm_pair_kernel<GATED, ROWPTR>, dim3(grid), dim3(mgb::Epi<GATED>::kThreads), mgb::pair_smem<GATED>(), stream, nullptr,
        tmA, tmBs, tmA4, offsets, E, MT / 2, K, rows_per_expert, half_rows, reinterpret_cast<__nv_bfloat16*>(out),
        ldo, balanced, row_ptr, nalign, rows_cap, cap_status, tma1_enabled());
  } else {
    if (const int rc = mgb_host::ensure_max_smem((const void*)mgb::moe_gemm_kernel<GATED, ROWPTR>,
                                                 mgb::gemm_smem<GATED>()))
      return rc;
    mgb_host::launch(mgb::moe_gemm_kernel<GATED, ROWPTR>, dim3(mgb_host::num_sms()), dim3(mgb::Epi<GATED>::kThreads), mgb::gemm_smem<GATED>(), stream, nullptr,
        tmA, tmB, offsets, E, MT, K, rows_per_expert, half_rows, reinterpret_cast<__nv_bfloat16*>(out), ldo, balanced,
        row_ptr, rows_cap, cap_status);
  }
  return mgb_host::launch_status();
}

// rows_per_unit: weight rows one CTA covers per unit (64 gated / 128 down); the pair kernel
// covers twice that per unit, so MT is given for the single-CTA tiling and halved here.
template <bool GATED>
int launch_moe_gemm(const void* w, int w_rows_total, const void* act, int act_rows, const int* offsets, int E,
                    int MT, int K, int rows_per_expert, int half_rows, void* out, int ldo, cudaStream_t stream,
                    const long long* row_ptr = nullptr) {
  const bool pair = use_pair_kernel() && MT % 2 == 0 && (mgb_host::num_sms() & ~1) >= 2;
  // token tiling: the gated GEMM balances its tiles (see token_tile); MGB_GEMM_BALANCED=0/1 overrides
  static const int bal_env = [] {
    const char* e = getenv("MGB_GEMM_BALANCED");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  const bool balanced = bal_env < 0 ? GATED : bal_env == 1;
  CUtensorMap tmA, tmB, tmA4 = {};
  mgb::BMaps tmBs;
  if (GATED && pair && encode_gate_up_4d(&tmA4, w, E, half_rows, K)) return MGB_ECUDA;
  if (mgb_host::encode_tmap_2d_bf16(&tmA, w, K, w_rows_total, (uint64_t)K * 2, mgb::kBK,
                                    GATED ? mgb::kBM / 2 : mgb::kBM) != CUDA_SUCCESS)
    return MGB_ECUDA;
  if (mgb_host::encode_tmap_2d_bf16(&tmB, act, K, act_rows, (uint64_t)K * 2, mgb::kBK, mgb::kBRows) != CUDA_SUCCESS)
    return MGB_ECUDA;
  if (pair && encode_bmaps(&tmBs, act, K, act_rows)) return MGB_ECUDA;
  if (row_ptr) {
    if (GATED) return MGB_EINVAL;  // only the down GEMM sends rows home
    return pair ? launch_variant<GATED, true, true>(tmA, tmA4, tmB, tmBs, offsets, E, MT, K, rows_per_expert, half_rows, out, ldo,
                                                   balanced, row_ptr, act_rows, stream)
                : launch_variant<GATED, false, true>(tmA, tmA4, tmB, tmBs, offsets, E, MT, K, rows_per_expert, half_rows, out, ldo,
                                                    balanced, row_ptr, act_rows, stream);
  }
  return pair ? launch_variant<GATED, true, false>(tmA, tmA4, tmB, tmBs, offsets, E, MT, K, rows_per_expert, half_rows, out, ldo,
                                                  balanced, nullptr, act_rows, stream)
              : launch_variant<GATED, false, false>(tmA, tmA4, tmB, tmBs, offsets, E, MT, K, rows_per_expert, half_rows, out, ldo,
                                                   balanced, nullptr, act_rows, stream);
}
}  // namespace

extern "C" {

// GEMM1 of the grouped expert FFN: h[r, :] = silu(x[r] W_g[e]^T) * (x[r] W_u[e]^T) for every
// permuted row r in expert e's segment [offsets[e], offsets[e+1]).
//   w_gate_up: [E, 2f, d] bf16 (HF MixtralExperts.gate_up_proj layout: gate rows then up rows)
//   x_perm:    [rows_cap, d] bf16, expert-major (output of mgb_permute)
//   h_out:     [rows_cap, f] bf16
int mgb_moe_gemm_gate_up(const void* w_gate_up, const void* x_perm, const int* offsets, int E, int d, int f,
                         int rows_cap, void* h_out, void* stream) {
  if (E < 1 || E > mgb::kMaxExperts || d % mgb::kBK || f % (mgb::kBM / 2) || rows_cap < 1) return MGB_EINVAL;
  return launch_moe_gemm<true>(w_gate_up, E * 2 * f, x_perm, rows_cap, offsets, E, f / (mgb::kBM / 2), d, 2 * f, f,
                               h_out, f, reinterpret_cast<cudaStream_t>(stream));
}

// GEMM2 of the grouped expert FFN: y[r, :] = h[r] W_d[e]^T.
//   w_down: [E, d, f] bf16 (HF MixtralExperts.down_proj layout), h: [rows_cap, f], y_out: [rows_cap, d]
int mgb_moe_gemm_down(const void* w_down, const void* h, const int* offsets, int E, int d, int f, int rows_cap,
                      void* y_out, void* stream) {
  if (E < 1 || E > mgb::kMaxExperts || f % mgb::kBK || d % mgb::kBM || rows_cap < 1) return MGB_EINVAL;
  return launch_moe_gemm<false>(w_down, E * d, h, rows_cap, offsets, E, d / mgb::kBM, f, d, 0, y_out, d,
                                reinterpret_cast<cudaStream_t>(stream));
}

// GEMM2 with the expert-parallel combine fused into the epilogue: output row r is written to
// row_ptr[r] (a UVA pointer into the source rank's y_perm, mgb_ep_row_ptrs; 0 = skip) instead of y.
int mgb_moe_gemm_down_ep(const void* w_down, const void* h, const int* offsets, int E, int d, int f, int rows_cap,
                         const long long* row_ptr, void* stream) {
  if (E < 1 || E > mgb::kMaxExperts || f % mgb::kBK || d % mgb::kBM || rows_cap < 1 || !row_ptr) return MGB_EINVAL;
  return launch_moe_gemm<false>(w_down, E * d, h, rows_cap, offsets, E, d / mgb::kBM, f, d, 0, nullptr, d,
                                reinterpret_cast<cudaStream_t>(stream), row_ptr);
}

// Trace read-out (MGB_GEMM_TRACE builds): copies g_ffn_trace [256][8] cycles and zeroes it.
int mgb_ffn_trace_read(long long* host_out) {
#ifdef MGB_GEMM_TRACE
  if (cudaMemcpyFromSymbol(host_out, mgb::g_ffn_trace, sizeof(mgb::g_ffn_trace)) != cudaSuccess) return MGB_ECUDA;
  static long long zero[256][8] = {};
  return cudaMemcpyToSymbol(mgb::g_ffn_trace, zero, sizeof(zero)) == cudaSuccess ? MGB_OK : MGB_ECUDA;
#else
  (void)host_out;
  return MGB_EINVAL;
#endif
}

// The whole expert FFN (gate/up + SiLU*up + down) as ONE persistent CTA-pair launch (moe_ffn_pair_kernel):
// the down units of expert e start as soon as e's h rows are complete, so the two GEMMs share one
// wave tail.  sync: 257 ints, zero before the first launch and left zero by every launch (per-expert
// completion counters + the exit ticket).  Shapes the pair tiling does not cover (f % 128, d % 256)
// or MGB_GEMM_PAIR=0 run the two grouped GEMMs back to back instead.
int mgb_moe_ffn(const void* w_gate_up, const void* w_down, const void* x_perm, const int* offsets, int E, int d, int f,
                int rows_cap, void* h_scratch, void* y_out, int* sync, void* stream) {
  if (E < 1 || E > mgb::kMaxExperts || d % mgb::kBM || f % (mgb::kBM / 2) || d % mgb::kBK || f % mgb::kBK ||
      rows_cap < 1 || !sync)
    return MGB_EINVAL;
  const bool fused = use_pair_kernel() && f % 128 == 0 && d % 256 == 0 && (mgb_host::num_sms() & ~1) >= 2;
  if (!fused) {
    const int rc = mgb_moe_gemm_gate_up(w_gate_up, x_perm, offsets, E, d, f, rows_cap, h_scratch, stream);
    return rc ? rc : mgb_moe_gemm_down(w_down, h_scratch, offsets, E, d, f, rows_cap, y_out, stream);
  }
  // K-blocked maps: a box covers kps consecutive 64-column K-blocks, one request per operand per stage.
  // kps = 1 (6 stages); MGB_FFN_KPS=2 takes 2 K-blocks per request in 3 stages of twice the size: half
  // the requests again, but slower (same box, Mixtral: 17.17 vs 16.84 ms per replayed forward) -- the
  // coarser ring costs more than the requests it saves once there are two per stage.
  static const int kps_env = [] {
    const char* e = getenv("MGB_FFN_KPS");
    return (e && e[0] == '2') ? 2 : 1;
  }();
  const int kps = (kps_env == 2 && (d / mgb::kBK) % 2 == 0 && (f / mgb::kBK) % 2 == 0) ? 2 : 1;
  CUtensorMap tAg, tAd;
  mgb::BMaps tBx, tBh;
  {
    const uint64_t dims[5] = {(uint64_t)mgb::kBK, (uint64_t)f, 2, (uint64_t)E, (uint64_t)d / mgb::kBK};
    const uint64_t strides[4] = {(uint64_t)d * 2, (uint64_t)f * d * 2, (uint64_t)2 * f * d * 2, (uint64_t)mgb::kBK * 2};
    const uint32_t box[5] = {(uint32_t)mgb::kBK, (uint32_t)mgb::kBM / 2, 2, 1, (uint32_t)kps};
    if (mgb_host::encode_tmap_bf16(&tAg, w_gate_up, 5, dims, strides, box, true, true) != CUDA_SUCCESS)
      return MGB_ECUDA;
  }
  {
    const uint64_t dims[3] = {(uint64_t)mgb::kBK, (uint64_t)E * d, (uint64_t)f / mgb::kBK};
    const uint64_t strides[2] = {(uint64_t)f * 2, (uint64_t)mgb::kBK * 2};
    const uint32_t box[3] = {(uint32_t)mgb::kBK, (uint32_t)mgb::kBM, (uint32_t)kps};
    if (mgb_host::encode_tmap_bf16(&tAd, w_down, 3, dims, strides, box, true, true) != CUDA_SUCCESS)
      return MGB_ECUDA;
  }
  if (encode_bmaps_kb(&tBx, x_perm, d, rows_cap, kps) || encode_bmaps_kb(&tBh, h_scratch, f, rows_cap, kps))
    return MGB_ECUDA;
  int* cap_status = mgb_host::capacity_status_ptr();
  if (!cap_status) return MGB_ECUDA;
  if (const int rc = mgb_host::ensure_max_smem((const void*)mgb::moe_ffn_pair_kernel, mgb::pair_smem<true>()))
    return rc;
  const mgb::FfnGemm gu{f / 128, d / mgb::kBK, 2 * f, f, f, reinterpret_cast<__nv_bfloat16*>(h_scratch)};
  const mgb::FfnGemm dn{d / 256, f / mgb::kBK, d, 0, d, reinterpret_cast<__nv_bfloat16*>(y_out)};
  static const int nalign = [] {
    const char* e = getenv("MGB_PAIR_NALIGN");
    return (e && atoi(e) == 32) ? 32 : 16;
  }();
  const int grid = mgb_host::num_sms() & ~1;
  mgb_host::launch(mgb::moe_ffn_pair_kernel, dim3(grid), dim3(mgb::Epi<true>::kThreads), mgb::pair_smem<true>(), reinterpret_cast<cudaStream_t>(stream), nullptr,
      tAg, tBx, tAd, tBh, offsets, E, gu, dn, nalign, rows_cap, cap_status, sync, kps);
  return mgb_host::launch_status();
}

// Both GEMMs back to back (h is caller-owned scratch [rows_cap, f]).
int mgb_grouped_ffn(const void* w_gate_up, const void* w_down, const void* x_perm, const int* offsets, int E, int d,
                    int f, int rows_cap, void* h_scratch, void* y_out, void* stream) {
  int rc = mgb_moe_gemm_gate_up(w_gate_up, x_perm, offsets, E, d, f, rows_cap, h_scratch, stream);
  if (rc != MGB_OK) return rc;
  return mgb_moe_gemm_down(w_down, h_scratch, offsets, E, d, f, rows_cap, y_out, stream);
}

}  // extern "C"
