// Router top-k, stable expert-major permutation, and weighted un-permute/combine (sm_100a).
//
// Replaces the ROUTER job of the module-based batching schedule
// (reference: pkg/src/moe_planner/offload_dag.py:418-425; cost hw_profile.py:273-275,291-292) and
// the implicit token grouping in front of the per-expert EXPERT_COMPUTE chunks
// (offload_dag.py:427-463).  Routing semantics follow HF transformers 5.5.0:
//   mode 0 (Mixtral, modeling_mixtral.py:109-116): logits = bf16(x W_g^T); p = softmax_fp32(logits);
//          top-k; w = p_sel / sum(p_sel).
//   mode 1 (DeepSeek-V2 greedy, modeling_deepseek_v2.py:100-105,125): logits = fp32(x) fp32(W_g)^T;
//          p = softmax_fp32; top-k; w = p_sel * routed_scaling_factor.
//   mode 2 (DeepSeek-V2 group_limited_greedy, :106-116): as mode 1 but experts restricted to the
//          top `topk_group` of `n_group` contiguous groups ranked by their max probability.
// Selection order is pinned (value descending, lower expert index first on ties) and is done on
// the logits (softmax is monotone), so indices are bit-exact given identical logits.
// The permutation is the stable sort of token-major flat entries (t*k + j) by expert
// (= HF grouped_mm's argsort with a stable tie rule, integrations/moe.py:368).
#include "common.cuh"

namespace mgb {

constexpr int kRouterTPB = 8;        // tokens per CTA
constexpr int kRouterThreads = 256;  // 8 warps: one token per warp in the selection phase
constexpr int kMaxE = 256;
constexpr int kMaxK = 8;
constexpr int kFusedScanMaxBlocks = 128;  // above this the column scan runs as its own E-CTA kernel

struct RouterArgs {
  const __nv_bfloat16* x;  // [T, d]
  const __nv_bfloat16* wg; // [E, d]
  const float* logits_in;  // optional [T, E]: skip the GEMV and route these logits
  int T, d, E, k, mode;
  float scaling;
  int n_group, topk_group;
  float* logits_out;       // optional [T, E]
  int* topk_idx;           // [T, k]
  float* topk_w;           // [T, k]
  int* local_rank;         // [T, k] rank of the entry among same-expert entries of its CTA
  int* block_hist;         // [nblk, E] -> converted in place to per-block exclusive bases
  int* counts;             // [E]
  int* offsets;            // [E+1]
  int* ticket;             // [1], zero on entry, reset to zero by the last CTA
};

// (value desc, index asc) ordering for selection
MGB_DEVINL bool better(float va, int ia, float vb, int ib) { return va > vb || (va == vb && ia < ib); }

MGB_DEVINL void warp_argbest(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (better(ov, oi, v, i)) { v = ov; i = oi; }
  }
}
MGB_DEVINL float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
MGB_DEVINL float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// GEMV = false: the logits come from the caller (a.logits_in); the kernel then carries none of the
// GEMV's registers (74 -> fewer per thread, so a DeepSeek-V2-Lite decode batch's 758 CTAs are one
// wave instead of 1.7)
template <bool GEMV>
__global__ void __launch_bounds__(kRouterThreads) router_topk_kernel(RouterArgs a) {
  mgb::pdl_enter();
  extern __shared__ __align__(16) uint8_t smem[];
  float* s_logit = reinterpret_cast<float*>(smem);                          // [TPB][E]
  int* s_exp = reinterpret_cast<int*>(s_logit + kRouterTPB * kMaxE);        // [TPB*k]
  __nv_bfloat16* s_x = reinterpret_cast<__nv_bfloat16*>(s_exp + kRouterTPB * kMaxK);  // [TPB][d]
  __shared__ bool s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * kRouterTPB;
  const int ntok = min(kRouterTPB, a.T - t0);
  const int E = a.E, d = a.d, k = a.k;

  // ---------------- phase 1: logits ----------------
  if (!GEMV) {
    // given fp32 logits (e.g. a cuBLAS bf16 GEMM with fp32 output); Mixtral's router linear is a
    // bf16 GEMM (modeling_mixtral.py:111), i.e. the fp32 accumulator rounded once to bf16
    for (int t = warp; t < ntok; t += kRouterThreads / 32)
      for (int e = lane; e < E; e += 32) {
        const float v = a.logits_in[(size_t)(t0 + t) * E + e];
        s_logit[t * kMaxE + e] = (a.mode == 0) ? bf16_round(v) : v;
      }
  } else if constexpr (GEMV) {
    // stage the CTA's (contiguous) token rows in smem with one bulk copy (TMA engine)
    const int vec_per_row = d / 8;
    __shared__ __align__(8) uint64_t s_bar;
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      fence_mbar_init();
      const uint32_t bytes = (uint32_t)ntok * d * 2;
      mbar_arrive_expect_tx(&s_bar, bytes);
      bulk_load(s_x, a.x + (size_t)t0 * d, bytes, &s_bar, policy_evict_first());
    }
    __syncthreads();
    mbar_wait(&s_bar, 0);
    for (int e = warp; e < E; e += kRouterThreads / 32) {
      float acc[kRouterTPB];
#pragma unroll
      for (int t = 0; t < kRouterTPB; ++t) acc[t] = 0.f;
      const uint4* wrow = reinterpret_cast<const uint4*>(a.wg + (size_t)e * d);
      // gate row in groups of 8 x 16 B per lane, all loads of a group in flight together; the
      // outer loop stays rolled to keep the kernel's code small (I-cache)
      constexpr int kWV = 8;
#pragma unroll 1
      for (int i0 = 0; i0 < vec_per_row; i0 += 32 * kWV) {
      uint4 wreg[kWV];
#pragma unroll
      for (int i = 0; i < kWV; ++i)
        if (i0 + lane + 32 * i < vec_per_row) wreg[i] = __ldg(wrow + i0 + lane + 32 * i);
#pragma unroll
      for (int i = 0; i < kWV; ++i) {
        const int c = i0 + lane + 32 * i;
        if (c >= vec_per_row) break;
        const uint4 w = wreg[i];
        const float w0 = bf16lo(w.x), w1 = bf16hi(w.x), w2 = bf16lo(w.y), w3 = bf16hi(w.y);
        const float w4 = bf16lo(w.z), w5 = bf16hi(w.z), w6 = bf16lo(w.w), w7 = bf16hi(w.w);
#pragma unroll
        for (int t = 0; t < kRouterTPB; ++t) {
          if (t < ntok) {
            const uint4 xv = reinterpret_cast<const uint4*>(s_x)[t * vec_per_row + c];
            float s = acc[t];
            s = fmaf(bf16lo(xv.x), w0, s); s = fmaf(bf16hi(xv.x), w1, s);
            s = fmaf(bf16lo(xv.y), w2, s); s = fmaf(bf16hi(xv.y), w3, s);
            s = fmaf(bf16lo(xv.z), w4, s); s = fmaf(bf16hi(xv.z), w5, s);
            s = fmaf(bf16lo(xv.w), w6, s); s = fmaf(bf16hi(xv.w), w7, s);
            acc[t] = s;
          }
        }
      }
      }
#pragma unroll
      for (int t = 0; t < kRouterTPB; ++t) {
        const float s = warp_sum(acc[t]);
        if (lane == 0 && t < ntok) s_logit[t * kMaxE + e] = (a.mode == 0) ? bf16_round(s) : s;
      }
    }
  }
  __syncthreads();

  // ---------------- phase 2: softmax + top-k (one warp per token) ----------------
  if (warp < ntok) {
    const int t = t0 + warp;
    const float* lg = s_logit + warp * kMaxE;
    if (a.logits_out)
      for (int e = lane; e < E; e += 32) a.logits_out[(size_t)t * E + e] = lg[e];
    float m = -INFINITY;
    for (int e = lane; e < E; e += 32) m = fmaxf(m, lg[e]);
    m = warp_max(m);
    float s = 0.f;
    for (int e = lane; e < E; e += 32) s += expf(lg[e] - m);
    s = warp_sum(s);
    const float inv = 1.0f / s;

    // group restriction (mode 2): allowed[e] via a bitmask over groups
    uint32_t group_ok = 0xffffffffu;
    if (a.mode == 2) {
      const int gsz = E / a.n_group;
      float gbest = -INFINITY;
      int gi = 0x7fffffff;
      if (lane < a.n_group) {
        gbest = -INFINITY;
        for (int e = lane * gsz; e < (lane + 1) * gsz; ++e) gbest = fmaxf(gbest, lg[e]);
        gi = lane;
      }
      group_ok = 0;
      for (int r = 0; r < a.topk_group; ++r) {
        float v = (group_ok >> lane) & 1u ? -INFINITY : gbest;
        int i = (group_ok >> lane) & 1u ? 0x7fffffff : gi;
        if (lane >= a.n_group) { v = -INFINITY; i = 0x7fffffff; }
        warp_argbest(v, i);
        group_ok |= 1u << i;
      }
    }
    // k rounds of warp arg-best over the (allowed, unselected) logits
    uint32_t taken[kMaxE / 32] = {0, 0, 0, 0, 0, 0, 0, 0};
    float psel[kMaxK];
    int isel[kMaxK];
    const int gsz = (a.mode == 2) ? E / a.n_group : E;
    for (int r = 0; r < k; ++r) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int e = lane, w = 0; e < E; e += 32, ++w) {
        if ((taken[w] >> lane) & 1u) continue;
        if (a.mode == 2 && !((group_ok >> (e / gsz)) & 1u)) continue;
        if (better(lg[e], e, bv, bi)) { bv = lg[e]; bi = e; }
      }
      warp_argbest(bv, bi);
      if ((bi & 31) == lane) taken[bi >> 5] |= 1u << lane;
      isel[r] = bi;
      psel[r] = expf(lg[bi] - m) * inv;
    }
    if (lane == 0) {
      float denom = 0.f;
      for (int r = 0; r < k; ++r) denom += psel[r];
      for (int r = 0; r < k; ++r) {
        a.topk_idx[(size_t)t * k + r] = isel[r];
        a.topk_w[(size_t)t * k + r] = (a.mode == 0) ? psel[r] / denom : psel[r] * a.scaling;
        s_exp[warp * k + r] = isel[r];
      }
    }
  }
  __syncthreads();

  // ---------------- phase 3: per-CTA histogram + stable local ranks ----------------
  const int nent = ntok * k;
  for (int i = threadIdx.x; i < nent; i += blockDim.x) {
    const int e = s_exp[i];
    int r = 0;
    for (int j = 0; j < i; ++j) r += (s_exp[j] == e);
    a.local_rank[(size_t)t0 * k + i] = r;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int c = 0;
    for (int j = 0; j < nent; ++j) c += (s_exp[j] == e);
    a.block_hist[(size_t)blockIdx.x * E + e] = c;
  }
  if ((int)gridDim.x > kFusedScanMaxBlocks) return;  // many blocks: router_scan_kernel finishes the job
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(a.ticket, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;

  // ---------------- last CTA: per-block bases, counts, offsets ----------------
  __threadfence();
  int* s_cnt = reinterpret_cast<int*>(smem);  // reuse
  // Exclusive scan of block_hist down each expert column.  A warp owns 4 experts at a time and
  // 32 blocks per chunk (all loads of a chunk in flight together, warp shuffles for the scan),
  // so the serial depth is nblk/32 L2 round trips instead of nblk.
  {
    const int NB = gridDim.x;
    for (int eg = warp; eg * 4 < E; eg += kRouterThreads / 32) {
      int carry[4] = {0, 0, 0, 0};
      for (int b0 = 0; b0 < NB; b0 += 32) {
        const int b = b0 + lane;
        int v[4];
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          const int e = eg * 4 + qd;
          v[qd] = (e < E && b < NB) ? __ldcg(a.block_hist + (size_t)b * E + e) : 0;
        }
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          int incl = v[qd];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          const int e = eg * 4 + qd;
          if (e < E && b < NB) a.block_hist[(size_t)b * E + e] = carry[qd] + incl - v[qd];
          carry[qd] += __shfl_sync(0xffffffffu, incl, 31);
        }
      }
      if (lane == 0)
        for (int qd = 0; qd < 4; ++qd) {
          const int e = eg * 4 + qd;
          if (e < E) {
            a.counts[e] = carry[qd];
            s_cnt[e] = carry[qd];
          }
        }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < E; ++e) {
      a.offsets[e] = run;
      run += s_cnt[e];
    }
    a.offsets[E] = run;
    *a.ticket = 0;
  }
}

// Column scan of the per-CTA expert histograms for large T: one CTA per expert turns its column
// into exclusive per-block bases (4 blocks per thread, warp shuffles + one smem pass per chunk of
// 1024 blocks) and writes counts[e]; the last CTA to finish derives offsets[E+1] from counts.
__global__ void __launch_bounds__(256) router_scan_kernel(int* __restrict__ block_hist, int nblk, int E,
                                                          int* __restrict__ counts, int* __restrict__ offsets,
                                                          int* __restrict__ ticket) {
  mgb::pdl_enter();
  const int e = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int s_warp[8];
  __shared__ int s_carry;
  __shared__ bool s_last;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < nblk; base += 256 * 4) {
    int v[4];
    const int b0 = base + tid * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (b0 + i < nblk) ? __ldcg(block_hist + (size_t)(b0 + i) * E + e) : 0;
    const int s = v[0] + v[1] + v[2] + v[3];
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += s_warp[w];
    int run = s_carry + wpre + incl - s;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (b0 + i < nblk) block_hist[(size_t)(b0 + i) * E + e] = run;
      run += v[i];
    }
    __syncthreads();
    if (tid == 255) s_carry = run;  // thread 255 holds the chunk's inclusive total
    __syncthreads();
  }
  if (tid == 0) counts[e] = s_carry;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(ticket, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // every expert's count in flight at once (a serial loop waited for E dependent L2 round trips)
  __shared__ int s_cnt[kMaxE];
  for (int i = tid; i < E; i += 256) s_cnt[i] = __ldcg(counts + i);
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int i = 0; i < E; ++i) {
      offsets[i] = run;
      run += s_cnt[i];
    }
    offsets[E] = run;
    *ticket = 0;
  }
}

// One warp per (token, slot) entry: compute the permuted row and copy x[t] there (16 B vectors).
template <int U>  // 16-byte vectors per lane held in flight (the launcher sizes it to the row)
__global__ void permute_kernel(const __nv_bfloat16* __restrict__ x, const int* __restrict__ topk_idx,
                               const int* __restrict__ local_rank, const int* __restrict__ block_base,
                               const int* __restrict__ offsets, int T, int d, int k, int E, int tpb,
                               __nv_bfloat16* __restrict__ x_perm, int* __restrict__ src_token,
                               int* __restrict__ dst_pos, const long long* __restrict__ peer_base,
                               const int* __restrict__ disp_row, int E_local, int recv_cap,
                               int* __restrict__ cap_status) {
  mgb::pdl_enter();
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= T * k) return;
  const int t = gw / k;
  const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)t * d);
  // the token's row (its first 512*U bytes) is requested before the routing lookups that place it, so the row
  // and the index chain (expert -> offsets / block base / rank) are in flight together
  const int nvec = d / 8;
  uint4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (lane + 32 * u < nvec) v[u] = ld_nc_v4(src + lane + 32 * u);
  const int e = topk_idx[gw];
  const int pos = offsets[e] + block_base[(size_t)(t / tpb) * E + e] + local_rank[gw];
  if (lane == 0) {
    dst_pos[gw] = pos;
    src_token[pos] = t;
  }
  // expert-parallel dispatch fused into the permutation: the row goes straight into the receive
  // buffer of the expert's owner rank (peer memory over NVLink), at this source's segment of expert e
  uint4* dst;
  if (peer_base) {
    const int row = disp_row[e] + pos - offsets[e];
    if (row < 0 || row >= recv_cap) {  // the owner's receive buffer is full: status, no write
      if (lane == 0 && atomicCAS(cap_status, 0, MGB_ECAPACITY) == 0) {
        cap_status[1] = row + 1;
        cap_status[2] = recv_cap;
        cap_status[3] = kCapDispatch;
      }
      return;
    }
    dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(peer_base[e / E_local]) + (size_t)row * d);
  } else {
    dst = reinterpret_cast<uint4*>(x_perm + (size_t)pos * d);
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (lane + 32 * u < nvec) dst[lane + 32 * u] = v[u];
  for (int c0 = lane + 32 * U; c0 < nvec; c0 += 32 * U) {  // rows wider than 512*U bytes
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + 32 * u < nvec) v[u] = ld_nc_v4(src + c0 + 32 * u);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + 32 * u < nvec) dst[c0 + 32 * u] = v[u];
  }
}

// out[t] = bf16( sum_j w[t,j] * y[dst[t,j]] ) (fp32, j ascending), then optional
//          moe = bf16(moe + shared[t]), then optional out = bf16(residual[t] + moe),
//          then optional norm_out[t] = RMSNorm(out[t]) * norm_w (HF MixtralRMSNorm rounding) --
//          the next layer's input norm fused into the row this CTA just produced.
// One CTA per token; the whole row lives in registers (<= kCombineVec 16 B vectors / thread).
constexpr int kCombineThreads = 256;
constexpr int kCombineVec = 4;  // d <= 8192
// One CTA per token; VEC 16-byte columns per thread (the launcher picks the smallest VEC that covers
// d, so registers -- and with them resident CTAs per SM -- follow the row width).  The token's
// residual / shared-expert rows are requested before its routing entries arrive, and all k expert
// rows of a column are in flight together: a CTA waits for two memory round trips, not four.
template <int VEC, int KMAX = kMaxK, int NTH = kCombineThreads>
__global__ void __launch_bounds__(NTH)
combine_kernel(const __nv_bfloat16* __restrict__ y_perm, const int* __restrict__ dst_pos,
               const float* __restrict__ topk_w, const __nv_bfloat16* __restrict__ shared_out,
               const __nv_bfloat16* residual, int T, int d, int k,
               __nv_bfloat16* out,  // may alias residual (in-place residual add)
               const __nv_bfloat16* __restrict__ norm_w, float eps, __nv_bfloat16* __restrict__ norm_out) {
  mgb::pdl_enter();
  const int t = blockIdx.x;
  __shared__ int s_pos[kMaxK];
  __shared__ float s_w[kMaxK];
  __shared__ float s_red[NTH / 32];
  const int nvec = d / 8;
  uint4 rv[VEC], sv[VEC];
#pragma unroll
  for (int u = 0; u < VEC; ++u) {  // routing-independent rows first (read before out is written)
    const int c = threadIdx.x + u * NTH;
    if (c < nvec) {
      if (residual) rv[u] = reinterpret_cast<const uint4*>(residual + (size_t)t * d)[c];
      if (shared_out) sv[u] = ld_nc_v4(reinterpret_cast<const uint4*>(shared_out + (size_t)t * d) + c);
    }
  }
  if (threadIdx.x < k) {
    s_pos[threadIdx.x] = dst_pos[(size_t)t * k + threadIdx.x];
    s_w[threadIdx.x] = topk_w[(size_t)t * k + threadIdx.x];
  }
  __syncthreads();
  float acc[VEC][8];
#pragma unroll
  for (int u = 0; u < VEC; ++u)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[u][i] = 0.f;
  // all k rows of a 16-byte column in flight at once (k independent loads per thread), then the fp32
  // weighted sum in j order (j ascending, as the oracle)
#pragma unroll
  for (int u = 0; u < VEC; ++u) {
    const int c = threadIdx.x + u * NTH;
    if (c < nvec) {
      uint4 v[KMAX];
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (j < k) v[j] = ld_nc_v4(reinterpret_cast<const uint4*>(y_perm + (size_t)s_pos[j] * d) + c);
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (j < k) {
          const float w = s_w[j];
          acc[u][0] += w * bf16lo(v[j].x); acc[u][1] += w * bf16hi(v[j].x);
          acc[u][2] += w * bf16lo(v[j].y); acc[u][3] += w * bf16hi(v[j].y);
          acc[u][4] += w * bf16lo(v[j].z); acc[u][5] += w * bf16hi(v[j].z);
          acc[u][6] += w * bf16lo(v[j].w); acc[u][7] += w * bf16hi(v[j].w);
        }
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < VEC; ++u) {
    const int c = threadIdx.x + u * NTH;
    if (c >= nvec) continue;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[u][i] = bf16_round(acc[u][i]);
    if (shared_out) {
      const float f[8] = {bf16lo(sv[u].x), bf16hi(sv[u].x), bf16lo(sv[u].y), bf16hi(sv[u].y),
                          bf16lo(sv[u].z), bf16hi(sv[u].z), bf16lo(sv[u].w), bf16hi(sv[u].w)};
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[u][i] = bf16_round(acc[u][i] + f[i]);
    }
    if (residual) {
      const float f[8] = {bf16lo(rv[u].x), bf16hi(rv[u].x), bf16lo(rv[u].y), bf16hi(rv[u].y),
                          bf16lo(rv[u].z), bf16hi(rv[u].z), bf16lo(rv[u].w), bf16hi(rv[u].w)};
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[u][i] = bf16_round(acc[u][i] + f[i]);
    }
    uint4 o;
    o.x = pack_bf16x2(acc[u][0], acc[u][1]); o.y = pack_bf16x2(acc[u][2], acc[u][3]);
    o.z = pack_bf16x2(acc[u][4], acc[u][5]); o.w = pack_bf16x2(acc[u][6], acc[u][7]);
    reinterpret_cast<uint4*>(out + (size_t)t * d)[c] = o;
#pragma unroll
    for (int i = 0; i < 8; ++i) ss = fmaf(acc[u][i], acc[u][i], ss);
  }
  if (!norm_out) return;
  // fused RMSNorm of the row just written (block reduction of the sum of squares); the norm weights
  // are requested before the reduction's barrier
  uint4 wv[VEC];
#pragma unroll
  for (int u = 0; u < VEC; ++u) {
    const int c = threadIdx.x + u * NTH;
    if (c < nvec) wv[u] = reinterpret_cast<const uint4*>(norm_w)[c];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < NTH / 32; ++i) tot += s_red[i];
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
#pragma unroll
  for (int u = 0; u < VEC; ++u) {
    const int c = threadIdx.x + u * NTH;
    if (c >= nvec) continue;
    const float wf[8] = {bf16lo(wv[u].x), bf16hi(wv[u].x), bf16lo(wv[u].y), bf16hi(wv[u].y),
                         bf16lo(wv[u].z), bf16hi(wv[u].z), bf16lo(wv[u].w), bf16hi(wv[u].w)};
    float r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = wf[i] * bf16_round(acc[u][i] * inv);
    uint4 o;
    o.x = pack_bf16x2(r[0], r[1]); o.y = pack_bf16x2(r[2], r[3]);
    o.z = pack_bf16x2(r[4], r[5]); o.w = pack_bf16x2(r[6], r[7]);
    reinterpret_cast<uint4*>(norm_out + (size_t)t * d)[c] = o;
  }
}

}  // namespace mgb

extern "C" {

// Number of router CTAs (= rows of the block_hist workspace) for T tokens.
int mgb_router_num_blocks(int T) { return (T + mgb::kRouterTPB - 1) / mgb::kRouterTPB; }
int mgb_router_tokens_per_block(void) { return mgb::kRouterTPB; }

// Fused router: gate GEMV (or given logits) -> softmax -> pinned-order top-k -> weights, plus
// per-expert counts/offsets and the per-CTA data the stable permutation needs.
int mgb_router_topk(const void* x, const void* w_gate, const float* logits_in, int T, int d, int E, int k,
                    int mode, float scaling, int n_group, int topk_group, float* logits_out, int* topk_idx,
                    float* topk_w, int* local_rank, int* block_hist, int* counts, int* offsets, int* ticket,
                    void* stream) {
  if (T < 1 || E < 1 || E > mgb::kMaxE || k < 1 || k > mgb::kMaxK || k > E || mode < 0 || mode > 2)
    return MGB_EINVAL;
  if (!logits_in && (d % 8 || d < 8)) return MGB_EINVAL;
  if (mode == 2 && (n_group < 1 || n_group > 32 || E % n_group || topk_group < 1 || topk_group > n_group ||
                    topk_group * (E / n_group) < k))
    return MGB_EINVAL;
  mgb::RouterArgs a{reinterpret_cast<const __nv_bfloat16*>(x), reinterpret_cast<const __nv_bfloat16*>(w_gate),
                    logits_in, T, d, E, k, mode, scaling, n_group, topk_group, logits_out, topk_idx, topk_w,
                    local_rank, block_hist, counts, offsets, ticket};
  const int nblk = mgb_router_num_blocks(T);
  const size_t smem = sizeof(float) * mgb::kRouterTPB * mgb::kMaxE + sizeof(int) * mgb::kRouterTPB * mgb::kMaxK +
                      (logits_in ? 0 : (size_t)mgb::kRouterTPB * d * 2);
  auto kern = logits_in ? mgb::router_topk_kernel<false> : mgb::router_topk_kernel<true>;
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return MGB_ECUDA;
  }
  mgb_host::launch(kern, dim3(nblk), dim3(mgb::kRouterThreads), smem, reinterpret_cast<cudaStream_t>(stream), nullptr,
      a);
  if (nblk > mgb::kFusedScanMaxBlocks)
    mgb_host::launch(mgb::router_scan_kernel, dim3(E), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
        block_hist, nblk, E, counts, offsets,
                                                                                   ticket);
  return mgb_host::launch_status();
}

// Stable expert-major permutation: x_perm[pos] = x[t] for every (t, j), pos = offsets[e] +
// block_base[t / tpb][e] + local_rank[t, j]; also src_token[pos] = t and dst_pos[t, j] = pos.
int mgb_permute(const void* x, const int* topk_idx, const int* local_rank, const int* block_base,
                const int* offsets, int T, int d, int k, int E, void* x_perm, int* src_token, int* dst_pos,
                void* stream) {
  if (T < 1 || d % 8 || k < 1 || k > mgb::kMaxK) return MGB_EINVAL;
  const int warps = T * k;
  const int threads = 256;
  const int blocks = (warps * 32 + threads - 1) / threads;
  mgb_host::launch((d <= 2048 ? mgb::permute_kernel<8> : mgb::permute_kernel<16>), dim3(blocks), dim3(threads), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(x), topk_idx, local_rank, block_base, offsets, T, d, k, E,
      mgb::kRouterTPB, reinterpret_cast<__nv_bfloat16*>(x_perm), src_token, dst_pos, nullptr, nullptr, 1, 0, nullptr);
  return mgb_host::launch_status();
}

// Expert-parallel dispatch fused with the permutation: row (t, j) of expert e = topk_idx[t, j] is
// written to peer_base[e / E_local] (the owner rank's receive buffer, a UVA peer pointer) at row
// disp_row[e] + (its position within expert e's segment).  dst_pos / src_token are the local
// permuted positions, as mgb_permute writes them (the combine on this rank uses them).  A row that
// would land at or past recv_rows_cap (the owner's fixed-capacity receive buffer) is not written;
// the overflow is recorded for mgb_capacity_status.
int mgb_ep_permute_dispatch(const void* x, const int* topk_idx, const int* local_rank, const int* block_base,
                            const int* offsets, int T, int d, int k, int E, int E_local, const long long* peer_base,
                            const int* disp_row, int recv_rows_cap, int* src_token, int* dst_pos, void* stream) {
  if (T < 1 || d % 8 || k < 1 || k > mgb::kMaxK || E_local < 1 || E % E_local || !peer_base || !disp_row ||
      recv_rows_cap < 1)
    return MGB_EINVAL;
  int* cap_status = mgb_host::capacity_status_ptr();
  if (!cap_status) return MGB_ECUDA;
  const int warps = T * k;
  const int threads = 256;
  const int blocks = (warps * 32 + threads - 1) / threads;
  mgb_host::launch((d <= 2048 ? mgb::permute_kernel<8> : mgb::permute_kernel<16>), dim3(blocks), dim3(threads), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(x), topk_idx, local_rank, block_base, offsets, T, d, k, E,
      mgb::kRouterTPB, nullptr, src_token, dst_pos, peer_base, disp_row, E_local, recv_rows_cap, cap_status);
  return mgb_host::launch_status();
}

// Destination of every row of the owner's expert-major receive buffer for the combine send: the
// rows are (local expert i, source s) segments in that order; segment j = i * W + s starts at
// seg_start[j] (ascending), holds seg_len[j] rows and maps row q to row q + seg_delta[j] of source
// s's y_perm, whose base is peer_base[s].  Rows past the last segment get 0 (skipped).
__global__ void ep_row_ptrs_kernel(const int* __restrict__ seg_start, const int* __restrict__ seg_len,
                                   const int* __restrict__ seg_delta, int n_seg, int W,
                                   const long long* __restrict__ peer_base, int row_bytes, int rows_cap,
                                   long long* __restrict__ row_ptr) {
  mgb::pdl_enter();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= rows_cap) return;
  int lo = 0, hi = n_seg - 1;  // last segment with start <= q
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_start[mid] <= q) lo = mid; else hi = mid - 1;
  }
  long long p = 0;
  if (seg_start[lo] <= q && q < seg_start[lo] + seg_len[lo])
    p = peer_base[lo % W] + (long long)(q + seg_delta[lo]) * row_bytes;
  row_ptr[q] = p;
}

int mgb_ep_row_ptrs(const int* seg_start, const int* seg_len, const int* seg_delta, int n_seg, int W,
                    const long long* peer_base, int row_bytes, int rows_cap, long long* row_ptr, void* stream) {
  if (n_seg < 1 || W < 1 || n_seg % W || row_bytes < 16 || rows_cap < 1) return MGB_EINVAL;
  mgb_host::launch(ep_row_ptrs_kernel, dim3((rows_cap + 255) / 256), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      seg_start, seg_len, seg_delta, n_seg, W, peer_base, row_bytes, rows_cap, row_ptr);
  return mgb_host::launch_status();
}

// Weighted un-permute + combine (fp32, j ascending, one bf16 rounding), optional shared-expert
// add and residual add (HF grouped_mm semantics, integrations/moe.py:417-429), optionally fused
// with the following RMSNorm (norm_w != NULL: norm_out = RMSNorm(out) * norm_w).
int mgb_unpermute_combine(const void* y_perm, const int* dst_pos, const float* topk_w, const void* shared_out,
                          const void* residual, int T, int d, int k, void* out, const void* norm_w, float eps,
                          void* norm_out, void* stream) {
  if (T < 1 || d % 8 || d > 8 * mgb::kCombineThreads * mgb::kCombineVec || k < 1 || k > mgb::kMaxK ||
      (norm_out && !norm_w))
    return MGB_EINVAL;
  const int vec = (d / 8 + mgb::kCombineThreads - 1) / mgb::kCombineThreads;
  auto kern = vec <= 1 ? mgb::combine_kernel<1> : vec <= 2 ? mgb::combine_kernel<2> : mgb::combine_kernel<mgb::kCombineVec>;
  int nth = mgb::kCombineThreads;
  if (k <= 2 && d / 8 <= 128 * 4 && d / 8 > 256) {
    // top-2 rows of a 2-4 k-wide row (Mixtral): 128 threads x 4 vectors and a k <= 2 register budget, so
    // a decode batch's CTAs are resident in one wave (256 x 2 with room for 8 rows: 80 registers, 3 CTAs
    // per SM, 1.9 waves at B = 827)
    kern = mgb::combine_kernel<4, 2, 128>;
    nth = 128;
  }
  mgb_host::launch(kern, dim3(T), dim3(nth), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(y_perm), dst_pos, topk_w,
      reinterpret_cast<const __nv_bfloat16*>(shared_out), reinterpret_cast<const __nv_bfloat16*>(residual), T, d,
      k, reinterpret_cast<__nv_bfloat16*>(out), reinterpret_cast<const __nv_bfloat16*>(norm_w), eps,
      reinterpret_cast<__nv_bfloat16*>(norm_out));
  return mgb_host::launch_status();
}

}  // extern "C"
