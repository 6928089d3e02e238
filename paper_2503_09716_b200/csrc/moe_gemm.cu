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
//   GEMM1 (mode 0): A = W_gu[e] rows {gate tile, up tile}, B = X_perm rows of expert e, K = d.
//                   Two TMEM accumulators (gate, up) so SiLU(gate)*up is formed per TMEM lane.
//   GEMM2 (mode 1): A = W_d[e] rows, B = H rows of expert e, K = f.
// Persistent grid (one CTA per SM), static round-robin over (expert, token-tile, row-tile) units
// ordered row-tile-fastest so concurrently running CTAs share the same token tile in L2.
// Warp roles: w0 = TMA producer, w1 = MMA issuer (+TMEM owner), w2..w5 = epilogue.
#include <cstdlib>

#include "common.cuh"

namespace mgb {

constexpr int kBM = 128;        // weight rows per tile (UMMA M)
constexpr int kBK = 64;         // K per stage (one 128 B swizzle row of bf16)
constexpr int kBNMax = 256;     // max tokens per tile (UMMA N)
constexpr int kBRows = 32;      // token rows per TMA box
constexpr int kATileBytes = kBM * kBK * 2;         // 16 KB
constexpr int kBTileBytes = kBNMax * kBK * 2;      // 32 KB
constexpr int kBBoxBytes = kBRows * kBK * 2;       // 4 KB
constexpr int kMaxExperts = 256;

template <int NA>
struct GemmCfg {
  static constexpr int kStageBytes = NA * kATileBytes + kBTileBytes;
  static constexpr int kStages = (NA == 2) ? 3 : 4;
  static constexpr int kAccCols = NA * kBNMax;              // TMEM cols per accumulator set
  static constexpr int kAccStages = 512 / kAccCols;          // 1 (NA=2) or 2 (NA=1)
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 1024 /*bars etc*/;
};

struct UnitSched {
  const int* s_prefix;  // [E+1] units before expert e (smem)
  int E, MT;
  __device__ void decode(int u, const int* offs, int& e, int& nt, int& mt, int& tok0, int& n) const {
    int lo = 0, hi = E - 1;  // last e with prefix[e] <= u
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s_prefix[mid] <= u) lo = mid; else hi = mid - 1;
    }
    e = lo;
    int local = u - s_prefix[e];
    nt = local / MT;
    mt = local - nt * MT;
    const int beg = offs[e], cnt = offs[e + 1] - beg;
    tok0 = beg + nt * kBNMax;
    n = min(kBNMax, cnt - nt * kBNMax);
  }
};

template <int NA>
__global__ void __launch_bounds__(192, 1)
moe_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const int* __restrict__ offsets, int E, int MT, int K, int rows_per_expert,
                int half_rows, __nv_bfloat16* __restrict__ out, int ldo, int prefetch) {
  using Cfg = GemmCfg<NA>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tiles = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + Cfg::kStages;
  uint64_t* tfull_bar = empty_bar + Cfg::kStages;
  uint64_t* tempty_bar = tfull_bar + Cfg::kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + Cfg::kAccStages);
  __shared__ int s_prefix[kMaxExperts + 1];

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;

  // unit prefix over experts: units(e) = ceil(n_e / BN) * MT
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      s_prefix[e] = acc;
      const int cnt = offsets[e + 1] - offsets[e];
      acc += ((cnt + kBNMax - 1) / kBNMax) * MT;
    }
    s_prefix[E] = acc;
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < Cfg::kAccStages; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = s_prefix[E];
  UnitSched sched{s_prefix, E, MT};
  const int KB = K / kBK;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      // optional L2 prefetch of the weight tiles `prefetch` k-blocks ahead of the TMA loads
      // (crossing into the CTA's next unit); measured slower on B200 at decode shapes -> off.
      auto prefetch_a = [&](int u, int kb) {
        int e2, nt2, mt2, tok2, n2;
        sched.decode(u, offsets, e2, nt2, mt2, tok2, n2);
        const int r0 = e2 * rows_per_expert + mt2 * kBM;
        tma_prefetch_2d(&tmA, kb * kBK, r0);
        if (NA == 2) tma_prefetch_2d(&tmA, kb * kBK, r0 + half_rows);
      };
      if (blockIdx.x < total)
        for (int kb = 0; kb < prefetch && kb < KB; ++kb) prefetch_a(blockIdx.x, kb);
      for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int e, nt, mt, tok0, n;
        sched.decode(u, offsets, e, nt, mt, tok0, n);
        const int nb = (n + kBRows - 1) / kBRows;
        const uint32_t bytes = NA * kATileBytes + nb * kBBoxBytes;
        const int arow0 = e * rows_per_expert + mt * kBM;
        const int u_next = u + gridDim.x;
        for (int kb = 0; kb < KB; ++kb) {
          if (prefetch > 0) {
            const int pf = kb + prefetch;
            if (pf < KB) prefetch_a(u, pf);
            else if (u_next < total && pf - KB < KB) prefetch_a(u_next, pf - KB);
          }
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], bytes);
          uint8_t* st = tiles + stage * Cfg::kStageBytes;
          tma_load_2d(st, &tmA, &full_bar[stage], kb * kBK, arow0, pol_w);
          if (NA == 2) tma_load_2d(st + kATileBytes, &tmA, &full_bar[stage], kb * kBK, arow0 + half_rows, pol_w);
          uint8_t* bt = st + NA * kATileBytes;
          for (int j = 0; j < nb; ++j)
            tma_load_2d(bt + j * kBBoxBytes, &tmB, &full_bar[stage], kb * kBK, tok0 + j * kBRows, pol_x);
          if (++stage == Cfg::kStages) { stage = 0; phase ^= 1; }
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
        const uint32_t d0 = tmem_base + acc * Cfg::kAccCols;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(tiles + stage * Cfg::kStageBytes);
          const uint64_t a0 = make_sdesc_sw128(st);
          const uint64_t a1 = make_sdesc_sw128(st + kATileBytes);
          const uint64_t b0 = make_sdesc_sw128(st + NA * kATileBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint32_t acc_flag = (kb | k) ? 1u : 0u;
            // +32 B per 16-element K step inside the 128 B swizzle row (desc units of 16 B)
            umma_bf16(d0, a0 + 2 * k, b0 + 2 * k, idesc, acc_flag);
            if (NA == 2) umma_bf16(d0 + kBNMax, a1 + 2 * k, b0 + 2 * k, idesc, acc_flag);
          }
          umma_commit(&empty_bar[stage]);
          if (++stage == Cfg::kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull_bar[acc]);
        if (++acc == Cfg::kAccStages) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ------------------------------ epilogue (warps 2..5) ------------------------------
    const uint32_t q = warp & 3;          // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;        // weight row within the 128-row tile
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
      int e, nt, mt, tok0, n;
      sched.decode(u, offsets, e, nt, mt, tok0, n);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tl = tmem_base + ((q * 32) << 16) + acc * Cfg::kAccCols;
      __nv_bfloat16* ocol = out + (size_t)tok0 * ldo + mt * kBM + row;
      for (int c0 = 0; c0 < n; c0 += 32) {
        uint32_t g[32];
        tmem_ld32(tl + c0, g);
        if (NA == 2) {
          uint32_t up[32];
          tmem_ld32(tl + kBNMax + c0, up);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (c0 + j < n) {
              const float gv = bf16_round(__uint_as_float(g[j]));
              const float uv = bf16_round(__uint_as_float(up[j]));
              const float sv = bf16_round(gv / (1.0f + expf(-gv)));
              ocol[(size_t)(c0 + j) * ldo] = __float2bfloat16_rn(sv * uv);
            }
          }
        } else {
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c0 + j < n) ocol[(size_t)(c0 + j) * ldo] = __float2bfloat16_rn(__uint_as_float(g[j]));
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == Cfg::kAccStages) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem_base);
}

}  // namespace mgb

// ------------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------------
namespace {
int gemm_prefetch_distance() {
  static int v = [] {
    const char* e = getenv("MGB_GEMM_PREFETCH");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int NA>
int launch_moe_gemm(const void* w, int w_rows_total, const void* act, int act_rows, const int* offsets,
                    int E, int MT, int K, int rows_per_expert, int half_rows, void* out, int ldo,
                    cudaStream_t stream) {
  using Cfg = mgb::GemmCfg<NA>;
  CUtensorMap tmA, tmB;
  if (mgb_host::encode_tmap_2d_bf16(&tmA, w, K, w_rows_total, (uint64_t)K * 2, mgb::kBK, mgb::kBM) != CUDA_SUCCESS)
    return MGB_ECUDA;
  if (mgb_host::encode_tmap_2d_bf16(&tmB, act, K, act_rows, (uint64_t)K * 2, mgb::kBK, mgb::kBRows) != CUDA_SUCCESS)
    return MGB_ECUDA;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(mgb::moe_gemm_kernel<NA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::kSmemBytes) != cudaSuccess)
      return MGB_ECUDA;
    attr_set = true;
  }
  const int grid = mgb_host::num_sms();
  mgb::moe_gemm_kernel<NA><<<grid, 192, Cfg::kSmemBytes, stream>>>(
      tmA, tmB, offsets, E, MT, K, rows_per_expert, half_rows,
      reinterpret_cast<__nv_bfloat16*>(out), ldo, gemm_prefetch_distance());
  return cudaGetLastError() == cudaSuccess ? MGB_OK : MGB_ECUDA;
}
}  // namespace

extern "C" {

// GEMM1 of the grouped expert FFN: h[r, :] = silu(x[r] W_g[e]^T) * (x[r] W_u[e]^T) for every
// permuted row r in expert e's segment [offsets[e], offsets[e+1]).
//   w_gate_up: [E, 2f, d] bf16 (HF MixtralExperts.gate_up_proj layout: gate rows then up rows)
//   x_perm:    [rows_cap, d] bf16, expert-major (output of mgb_permute)
//   h_out:     [rows_cap, f] bf16
int mgb_moe_gemm_gate_up(const void* w_gate_up, const void* x_perm, const int* offsets, int E,
                         int d, int f, int rows_cap, void* h_out, void* stream) {
  if (E < 1 || E > mgb::kMaxExperts || d % mgb::kBK || f % mgb::kBM || rows_cap < 1) return MGB_EINVAL;
  return launch_moe_gemm<2>(w_gate_up, E * 2 * f, x_perm, rows_cap, offsets, E, f / mgb::kBM, d, 2 * f, f,
                            h_out, f, reinterpret_cast<cudaStream_t>(stream));
}

// GEMM2 of the grouped expert FFN: y[r, :] = h[r] W_d[e]^T.
//   w_down: [E, d, f] bf16 (HF MixtralExperts.down_proj layout), h: [rows_cap, f], y_out: [rows_cap, d]
int mgb_moe_gemm_down(const void* w_down, const void* h, const int* offsets, int E, int d, int f,
                      int rows_cap, void* y_out, void* stream) {
  if (E < 1 || E > mgb::kMaxExperts || f % mgb::kBK || d % mgb::kBM || rows_cap < 1) return MGB_EINVAL;
  return launch_moe_gemm<1>(w_down, E * d, h, rows_cap, offsets, E, d / mgb::kBM, f, d, 0, y_out, d,
                            reinterpret_cast<cudaStream_t>(stream));
}

// Both GEMMs back to back (h is caller-owned scratch [rows_cap, f]).
int mgb_grouped_ffn(const void* w_gate_up, const void* w_down, const void* x_perm, const int* offsets,
                    int E, int d, int f, int rows_cap, void* h_scratch, void* y_out, void* stream) {
  int rc = mgb_moe_gemm_gate_up(w_gate_up, x_perm, offsets, E, d, f, rows_cap, h_scratch, stream);
  if (rc != MGB_OK) return rc;
  return mgb_moe_gemm_down(w_down, h_scratch, offsets, E, d, f, rows_cap, y_out, stream);
}

}  // extern "C"
