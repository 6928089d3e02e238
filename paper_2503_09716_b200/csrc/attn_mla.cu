// Absorbed multi-head latent attention (DeepSeek-V2) decode on sm_100a — the ATTN_MECH_GPU job
// for MLA models (reference: pkg/src/moe_planner/offload_dag.py:393-402; the reference models
// DSV2's mechanism via an inflated activation, model_catalog.py:242-295).
//
// HF transformers 5.5.0 DeepseekV2Attention (modeling_deepseek_v2.py:337-396) up-projects the
// latent into per-head K/V.  This kernel computes the mathematically equal absorbed form
//     s_h(t) = (q_lat_h . c_t + q_pe_h . kpe_t) * scale,   o_lat_h = sum_t softmax(s_h)_t c_t
// with q_lat_h = W_UK_h^T q_nope_h and o_h = W_UV_h o_lat_h done by the caller (cuBLAS bmm), so
// the cache holds only the 576-wide latent row per token (1,152 B instead of 2*H*... per head).
// Equal to HF within bf16 tolerance, not bit-exact (different rounding points).
//
// Latent cache: pages of kMlaPage = 56 tokens stored exactly as the tensor cores read them from
// shared memory: 64-dim blocks [(R+r)/64][56 tok][128 B], each 128-byte token row holding its 8
// 16-byte chunks in 128B-swizzled order (chunk c of token t at position c ^ (t & 7)).  That one
// layout is, without any re-staging, both operands a page is used as:
//   S^T[64 tok, 16 heads] = C[64 tok, R+r] . Q^T          (A = page, K-major, SWIZZLE_128B)
//   O^T[R, 16 heads]     += C[:, :R]^T [R, 64 tok] . P^T  (A = page, MN-major, SWIZZLE_128B)
// The MMAs are 64 tokens tall; rows 56-63 are "phantom" rows that alias the next 64-dim block
// (masked to P = 0).  56-token pages let three stages (189 KB) fit in shared memory, which keeps
// enough bytes in flight per SM while a page is held for S^T -> softmax -> P.V.  The swizzle keeps
// the tensor cores' shared-memory reads conflict free; R + r is padded to a multiple of 64 in the
// page, and the append kernels write the padding of every token row as zeros: P.V's phantom rows
// (tokens 56-63 of a 64-dim block alias the next block's first 8 token rows) multiply P = 0 by those
// rows, padding included, so they must be finite.  Rows past a sequence's length may hold anything
// (masked from S, zeroed in shared memory before P.V).
// A page is one contiguous cp.async.bulk, and both GEMMs run on tcgen05 with fp32 accumulators in
// TMEM ("swap-AB": tokens / latent dims fill the MMA M side, the 16 heads of a work item are N).
//
// Persistent kernel, one CTA per SM, 10 warps:
//   warp 8  producer: streams the pages of every work item through a 3-stage smem ring, and Q
//   warp 9  MMA issuer (one elected lane): S^T of each page and P.V of each softmaxed page, issued
//           as each becomes ready (double-buffered TMEM accumulators)
//   warps 0-7 softmax + correction, two groups of four (heads 0-7, heads 8-15): TMEM -> registers
//           (lane = token), per-head online softmax with a warp transpose-reduction, P^T -> smem,
//           O accumulated in registers (lane = latent dim)
// A work item is (sequence, 16-head group); heads >= H are zero rows of Q and never stored.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

// S^T partial accumulators (k-step k -> partial k % SACC, summed by the softmax warps).  One: the
// softmax warps -- the kernel's bottleneck at the power-capped clocks of a long decode run -- then
// load and add a quarter of the TMEM columns; the single 36-MMA chain is hidden behind the other
// pages in flight (DSV2-Lite forward 59.5 -> 56.0 ms in the replayed graph vs 4 partials, same box).
#ifndef MGB_MLA_SACC
#define MGB_MLA_SACC 1
#endif

namespace mgb {

#ifndef MGB_MLA_PAGE
#define MGB_MLA_PAGE 56
#endif
#ifndef MGB_MLA_STAGES
#define MGB_MLA_STAGES 3
#endif
constexpr int kMlaPage = MGB_MLA_PAGE;     // tokens per latent page (swizzle atoms of 8 tokens)
constexpr int kMlaTile = 64;     // M of the S^T MMA / K of P.V: a page plus 8 phantom rows
constexpr int kMlaStages = MGB_MLA_STAGES;  // pages in flight per SM (3 x 63 KB for R = 512)
static_assert(kMlaPage % 8 == 0 && kMlaPage <= 64, "latent page = whole swizzle atoms within one MMA tile");
static_assert(kMlaStages <= 8, "the MMA issuer's page ring holds 8 pages between S^T and P.V");
constexpr int kMlaHeads = 16;    // heads per work item = N of both MMAs
constexpr int kMlaThreads = 320;  // 8 softmax warps + producer + MMA issuer

// Optional per-page timeline of CTA 0 (build with -DMGB_MLA_TRACE; tools/mla_trace.py):
// trace[ev * kTraceN + page] = %globaltimer (ns) of event ev for the CTA's page number `page`.
#ifdef MGB_MLA_TRACE
constexpr int kTraceN = 256;
__device__ unsigned long long g_mla_trace[16 * kTraceN];
MGB_DEVINL void mla_trace(int ev, int page) {
  if (blockIdx.x == 0 && page < kTraceN) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_mla_trace[ev * kTraceN + page] = t;
  }
}
#else
MGB_DEVINL void mla_trace(int, int) {}
#endif

// named barrier of one softmax warp group (ids 1, 2; 128 threads); 0 is __syncthreads
MGB_DEVINL void grp_bar(int grp) { asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory"); }
// the same barrier, returning whether any thread of the group passed true
MGB_DEVINL bool grp_bar_or(int grp, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred pi, po;\n\tsetp.ne.u32 pi, %1, 0;\n\tbar.red.or.pred po, %2, 128, pi;\n\t"
      "selp.u32 %0, 1, 0, po;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(1 + grp)
      : "memory");
  return r != 0;
}
// A page whose scores all stay within 2^kMlaSlack of their heads' running max takes the fast path:
// one barrier-with-OR instead of the max exchange (P <= 2^kMlaSlack stays exact to bf16 rounding,
// and fp32 l / O have the range).  Any score beyond it (always the item's first page) takes the
// exchange, which raises each head's max to its page max where that exceeds it by 2^8.
#ifndef MGB_MLA_SLACK
#define MGB_MLA_SLACK 32
#endif

template <int R, int RP>  // latent width, rope width
struct MlaCfg {
  static constexpr int D = R + RP;                         // cached row width
  static constexpr int NKB = (D + 63) / 64;                // 64-dim blocks per page (padded)
  static constexpr int kBlockBytes = kMlaPage * 128;       // one 64-dim block of a page
  static constexpr int kPageBytes = NKB * kBlockBytes;     // [NKB][56 tok][128 B swizzled]
  static constexpr int kQBlockBytes = kMlaHeads * 128;     // one 64-dim block of Q
  static constexpr int kQBytes = NKB * kQBlockBytes;       // [NKB][16 heads][128 B swizzled]
  static constexpr int kChunkBytes = kMlaTile * 16;        // P^T: [2 head groups][64 tok][8 heads]
  static constexpr int kPBytes = 2 * kMlaTile * 16;
  static constexpr int MT = R / 128;                       // O^T M tiles of 128 latent dims
  static constexpr int KS = D / 16;                        // k-steps of S^T
  // Small MMAs accumulating into one TMEM tile serialise on their latency, so S^T is split over
  // kSAcc independent partial accumulators (k-step k -> partial k % kSAcc, summed by the softmax
  // warps) and the P.V MMAs interleave their MT independent M tiles.
  static constexpr int kSAcc = KS % MGB_MLA_SACC == 0 ? MGB_MLA_SACC : (KS % 2 == 0 ? 2 : 1);
  static constexpr uint32_t kSCol = 0;                        // S^T: 2 buffers x kSAcc x 16 columns
  static constexpr uint32_t kOCol = 2 * kSAcc * 16;           // O^T: 2 buffers x MT x 16 columns
  static constexpr uint32_t kTmemCols = kOCol + 2 * MT * 16 <= 128 ? 128 : 256;
  static_assert(kOCol + 2 * MT * 16 <= 256, "TMEM budget");
  static constexpr int kOffQ = kMlaStages * kPageBytes;
  static constexpr int kOffP = kOffQ + kQBytes;
  static constexpr int kOffRed = kOffP + 2 * kPBytes;      // float [2][4][16] max + [4][16] sum
  static constexpr int kOffBar = kOffRed + 3 * 4 * 16 * 4;
  static constexpr int kBars = 3 * kMlaStages + 12;  // + per-stage cluster-empty barriers (multicast)
  static constexpr size_t kSmem = kOffBar + kBars * 8 + 16;
  static_assert(R % 128 == 0 && RP % 16 == 0 && kBlockBytes % 1024 == 0, "MLA shape");
  static_assert(kSmem <= 227 * 1024, "MLA smem");
};

// Reduce 8 per-head values over the 16 lanes of each half-warp (max or sum); afterwards lane l holds
// head (l >> 1) & 7 (both lanes of a pair agree).  7 shuffles by halving, then one pairwise step.
template <bool kMax>
MGB_DEVINL float xreduce8(float (&v)[8], int lane) {
#pragma unroll
  for (int o = 8; o >= 2; o >>= 1) {
    const bool hi = lane & o;
    const int half = o >> 1;  // 8 values -> 4 -> 2 -> 1
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float keep = hi ? v[i + half] : v[i];
      const float send = hi ? v[i] : v[i + half];
      const float got = __shfl_xor_sync(0xffffffffu, send, o);
      v[i] = kMax ? fmaxf(keep, got) : keep + got;
    }
  }
  const float got = __shfl_xor_sync(0xffffffffu, v[0], 1);
  return kMax ? fmaxf(v[0], got) : v[0] + got;
}

template <int R, int RP>
__global__ void __launch_bounds__(kMlaThreads, 1)
decode_attn_mla_kernel(const __grid_constant__ CUtensorMap tm_qlat,  // q_lat [H, B, R] as [64][H][R/64][B]
                       const __grid_constant__ CUtensorMap tm_qpe,   // q_pe [B, H, RP] as [RP][H][B]
                       const __nv_bfloat16* __restrict__ cache,      // latent pages
                       const int* __restrict__ block_table, int max_pages, const int* __restrict__ seq_lens,
                       int B, int H, float scale_log2, __nv_bfloat16* __restrict__ o_lat,  // [H, B, R]
                       int pf_dist, int cl) {
  mgb::pdl_enter();
  using C = MlaCfg<R, RP>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* pages = smem;
  uint8_t* q_s = smem + C::kOffQ;
  uint8_t* p_s = smem + C::kOffP;
  float* red = reinterpret_cast<float*>(smem + C::kOffRed);  // [2][4][16]
  float* lred = red + 2 * 4 * 16;                              // [4][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  constexpr int S = kMlaStages;
  uint64_t *full = bars, *empty = bars + S, *qfull = bars + 2 * S, *qempty = bars + 2 * S + 1,
           *sfull = bars + 2 * S + 2, *sempty = bars + 2 * S + 4, *pfull = bars + 2 * S + 6, *ofull = bars + 2 * S + 8,
           *oempty = bars + 2 * S + 10, *cempty = bars + 2 * S + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_hg = (H + kMlaHeads - 1) / kMlaHeads;
  const int n_items = B * n_hg;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMlaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&cempty[s], cl);  // (the leader's are used: every CTA of the cluster freed stage s)
    }
    mbar_init(qfull, 1);
    mbar_init(qempty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 8);
      mbar_init(&pfull[s], 8);
      mbar_init(&ofull[s], 1);
      mbar_init(&oempty[s], 8);
    }
    fence_mbar_init();
  }
  if (warp == 9) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if (cl > 1) cluster_sync();  // peers' barriers initialised before any remote arrive / multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ------------------------------ producer ------------------------------
    // lane 0 streams pages through the 3-stage ring; lane 1 refills the single Q buffer as soon as
    // the previous item's last S^T has consumed it (the two lanes wait independently).
    if (lane == 0) {
      // Cluster of cl CTAs = the cl head groups of one sequence (cl == n_hg): the leader streams each
      // page ONCE and multicasts it into every CTA's stage (the latent is read once per sequence, not
      // once per head group); each CTA arms its own full barrier and tells the leader its stage is
      // free.  Pages are read once: stream them past L2 (unless unclustered head groups share them).
      const bool mc = cl > 1;
      const bool leader = !mc || cluster_ctarank() == 0;
      const uint16_t mask = (uint16_t)((1u << cl) - 1);
      const uint32_t cempty_leader = mc ? mapa_shared(smem_u32(cempty), 0) : 0u;
      const uint64_t pol = (n_hg == 1 || mc) ? policy_evict_first() : policy_evict_last();
      // L2 prefetch cursor running pf_dist pages ahead of the smem ring
      int pf_it = blockIdx.x, pf_p = 0;
      auto prefetch_next = [&]() {
        while (pf_it < n_items) {
          const int pb = pf_it / n_hg;
          if (pf_p < (seq_lens[pb] + kMlaPage - 1) / kMlaPage) {
            bulk_prefetch_l2(cache + (size_t)block_table[(size_t)pb * max_pages + pf_p] * (C::kPageBytes / 2),
                             C::kPageBytes);
            ++pf_p;
            return;
          }
          pf_it += gridDim.x;
          pf_p = 0;
        }
      };
      if (leader)
        for (int i = 0; i < pf_dist; ++i) prefetch_next();
      int g = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int b = it / n_hg;
        const int np = (seq_lens[b] + kMlaPage - 1) / kMlaPage;
        const int* bt = block_table + (size_t)b * max_pages;
        for (int p = 0; p < np; ++p, ++g) {
          const int s = g % kMlaStages;
          mbar_wait(&empty[s], ((g / kMlaStages) & 1) ^ 1);
          mla_trace(0, g);  // 0: stage free, page load issued
          const int rows = min(kMlaPage, seq_lens[b] - p * kMlaPage);
          const __nv_bfloat16* src = cache + (size_t)bt[p] * (C::kPageBytes / 2);
          // a sequence's last, partial page: only its valid token rows of every 64-dim block (rows past
          // the end keep stale finite data; the softmax warps mask them and zero them before P.V)
          mbar_arrive_expect_tx(&full[s], rows == kMlaPage ? C::kPageBytes : C::NKB * rows * 128);
          if (mc) {
            mbar_arrive_cluster(cempty_leader + s * 8);
            if (!leader) continue;
            mbar_wait(&cempty[s], (g / kMlaStages) & 1);
          }
          prefetch_next();
          if (rows == kMlaPage) {
            if (mc) bulk_load_multicast(pages + s * C::kPageBytes, src, C::kPageBytes, &full[s], mask, pol);
            else bulk_load(pages + s * C::kPageBytes, src, C::kPageBytes, &full[s], pol);
          } else {
            for (int kb = 0; kb < C::NKB; ++kb) {
              uint8_t* dst = pages + s * C::kPageBytes + kb * C::kBlockBytes;
              const __nv_bfloat16* gsrc = src + kb * (C::kBlockBytes / 2);
              if (mc) bulk_load_multicast(dst, gsrc, rows * 128, &full[s], mask, pol);
              else bulk_load(dst, gsrc, rows * 128, &full[s], pol);
            }
          }
        }
      }
    } else if (lane == 1) {
      prefetch_tmap(&tm_qlat);
      prefetch_tmap(&tm_qpe);
      int qi = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int b = it / n_hg, hg = it - b * n_hg;
        if (seq_lens[b] <= 0) continue;
        // Q of the group -> [block][16 heads][128 B swizzled] (heads >= H and rope dims past RP
        // are zero-filled out of bounds)
        mbar_wait(qempty, (qi & 1) ^ 1);
        mbar_arrive_expect_tx(qfull, C::kQBytes);
        tma_load_4d(q_s, &tm_qlat, qfull, 0, hg * kMlaHeads, 0, b);
        for (int kb = R / 64; kb < C::NKB; ++kb)
          tma_load_3d(q_s + kb * C::kQBlockBytes, &tm_qpe, qfull, (kb - R / 64) * 64, hg * kMlaHeads, b);
        ++qi;
      }
    }
  } else if (warp == 9) {
    // ------------------------------ MMA issuer ------------------------------
    // Two independent in-order streams: S^T of page g needs page g in smem; P.V of page t needs
    // the softmax warps' P_t.  The warp polls both and issues whichever is ready, so a late page
    // never holds back the P.V (and with it the stage release) of the page before it.  The whole
    // warp runs this converged (warp-uniform conditions) so the MMAs issue back to back.
    const uint32_t idesc_s = make_idesc_bf16(64, kMlaHeads);
    const uint32_t idesc_o = make_idesc_bf16(128, kMlaHeads) | kIdescAMajorMN | kIdescBMajorMN;
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t pages_a = smem_u32(pages), q_a = smem_u32(q_s), p_a = smem_u32(p_s);
    // descriptors of stage / buffer 0; other stages and k-steps are constant offsets added to the
    // 14-bit start-address field (smem addresses < 256 KB never carry out of it)
    const uint64_t dC_s = make_sdesc_sw128(pages_a);                          // page as K-major A
    const uint64_t dC_o = make_sdesc_sw128_mn(pages_a, C::kBlockBytes, 1024);  // page as MN-major A
    const uint64_t dQ = make_sdesc_sw128(q_a);
    const uint64_t dP = make_sdesc_noswz(p_a, 128, C::kChunkBytes);
    int gs = 0, gpv = 0;            // next page for S^T / for P.V (global page counters)
    int it = blockIdx.x, p = 0, np = -1, qi = 0;  // S^T cursor: item, page in item
    int items_s = 0;                // items whose S^T stream has started (O buffer = item parity)
    // per page in flight between S^T and P.V: bit 0 = first page of its item, bit 1 = O buffer, bits
    // 2+ = the item's O-buffer use count (for the oempty phase)
    int ring[8];
    bool s_done = false;
    while (true) {
      if (!s_done && np < 0) {  // advance the S^T cursor to the next item with pages
        while (it < n_items) {
          np = __shfl_sync(0xffffffffu, (seq_lens[it / n_hg] + kMlaPage - 1) / kMlaPage, 0);
          if (np > 0) break;
          it += gridDim.x;
        }
        if (it >= n_items) s_done = true;
        p = 0;
      }
      const int sb = gs & 1, pb = gpv & 1;                       // TMEM S / P buffers
      const int sst = gs % kMlaStages, pst = gpv % kMlaStages;  // smem stages
      const bool can_s = !s_done && gs - gpv < 8 &&
                         __all_sync(0xffffffffu, mbar_test(&full[sst], (gs / kMlaStages) & 1) &&
                                                     mbar_test(&sempty[sb], ((gs >> 1) & 1) ^ 1) &&
                                                     mbar_test(qfull, qi & 1));
      bool can_pv = false;
      int rg = 0;
      if (gpv < gs) {
        rg = ring[gpv & 7];
        const int ob = (rg >> 1) & 1, use = rg >> 2;
        // the first P.V of an item overwrites its O buffer: the softmax warps must have read the
        // item that used it before (two items ago)
        can_pv = __all_sync(0xffffffffu, mbar_test(&pfull[pb], (gpv >> 1) & 1) &&
                                             (!(rg & 1) || mbar_test(&oempty[ob], (use & 1) ^ 1)));
      }
      if (can_pv) {  // O^T[ob] (+)= C_gpv[:, :R]^T . P_gpv^T (accumulated over the item's pages in TMEM)
        if (lane == 0) mla_trace(2, gpv);  // 2: P.V issued
        tc_fence_after();
        const int ob = (rg >> 1) & 1;
        const uint32_t first = rg & 1;
        const uint64_t a0 = dC_o + ((uint32_t)(pst * C::kPageBytes) >> 4), b0 = dP + ((uint32_t)(pb * C::kPBytes) >> 4);
        const uint32_t d0 = tm + C::kOCol + ob * C::MT * 16;
#pragma unroll
        for (int k = 0; k < kMlaTile / 16; ++k)
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt)
            umma_bf16_warp(d0 + mt * 16, a0 + ((mt * 2 * C::kBlockBytes + k * 2048) >> 4), b0 + ((k * 256) >> 4),
                           idesc_o, (k > 0 || !first) ? 1u : 0u);
        umma_commit_warp(&ofull[pb]);
        umma_commit_warp(&empty[pst]);
        ++gpv;
      } else if (can_s) {  // S^T[sb] = C_gs . Q^T over kSAcc partial accumulators
        if (lane == 0) mla_trace(1, gs);  // 1: page landed (+ S buffer free): S issued
        tc_fence_after();
        const uint64_t a0 = dC_s + ((uint32_t)(sst * C::kPageBytes) >> 4);
        const uint64_t b0 = dQ;
        const uint32_t d = tm + C::kSCol + sb * C::kSAcc * 16;
#pragma unroll
        for (int k = 0; k < C::KS; ++k)
          umma_bf16_warp(d + (k % C::kSAcc) * 16, a0 + (((k >> 2) * C::kBlockBytes + (k & 3) * 32) >> 4),
                         b0 + (((k >> 2) * C::kQBlockBytes + (k & 3) * 32) >> 4), idesc_s, k >= C::kSAcc);
        umma_commit_warp(&sfull[sb]);
        ring[gs & 7] = (p == 0 ? 1 : 0) | ((items_s & 1) << 1) | ((items_s >> 1) << 2);
        ++gs;
        if (++p == np) {  // last page of the item: its Q buffer may be refilled
          umma_commit_warp(qempty);
          ++qi;
          ++items_s;
          it += gridDim.x;
          np = -1;
        }
      } else if (s_done && gpv == gs) {
        break;
      }
    }
  } else {
    // ------------------------- softmax + correction -------------------------
    // Eight warps: warp w reads TMEM lane quarter w % 4 (tokens 16*(w%4) .. +15 of the page) for the
    // eight heads of group w / 4.  Heads are independent, so the two groups never combine state;
    // splitting them halves every warp's per-page softmax chain and puts two warps on each
    // scheduler to hide its latencies.
    constexpr int HG = kMlaHeads / 2;  // heads per warp group
    const int q = warp & 3, grp = warp >> 2;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t col0 = grp * HG;     // first TMEM column of the group's heads in S / O tiles
    float* gred = red;  // [2][4][16] row maxima; this group owns heads [col0, col0 + HG)
    int g = 0;
    int items_sm = 0;  // items with pages processed (O buffer = parity)
    int pvw = 0;       // P.V completions (ofull phases) consumed, in page order
    // ofull[g & 1] completes once per page; waiting for every phase in order keeps the parity waits
    // unambiguous (the MMA can never be two phases ahead of pvw: P.V(g) needs P(g) first)
    auto wait_pv_upto = [&](int G) {
      while (pvw <= G) {
        mbar_wait(&ofull[pvw & 1], (pvw >> 1) & 1);
        ++pvw;
      }
    };
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int b = it / n_hg, hg = it - b * n_hg;
      const int len = seq_lens[b];
      if (threadIdx.x == 0) mla_trace(12, g);  // 12: next item's length loaded
      const int np = (len + kMlaPage - 1) / kMlaPage;
      if (np == 0) {
        for (int i = threadIdx.x; i < kMlaHeads * R; i += 256) {
          const int h = hg * kMlaHeads + i / R;
          if (h < H) o_lat[((size_t)h * B + b) * R + i % R] = __float2bfloat16_rn(0.f);
        }
        continue;
      }
      // Online softmax with the O accumulator resident in TMEM (the P.V MMAs accumulate over the
      // item's pages): the running max a head's P is computed against is only raised when a page's
      // max exceeds it by more than 2^8 (P <= 256 is exact enough in bf16 and fp32), so the O
      // rescale (TMEM load, scale, store) happens on a handful of pages per item, not every page.
      const int ob = items_sm & 1;
      float m_used[HG], lpart[HG];
#pragma unroll
      for (int h = 0; h < HG; ++h) {
        m_used[h] = -INFINITY;
        lpart[h] = 0.f;
      }
      const uint32_t ocol = C::kOCol + ob * C::MT * 16 + col0;
      for (int p = 0; p < np; ++p, ++g) {
        const int s = g & 1, st = g % kMlaStages;
        const int n = min(kMlaPage, len - p * kMlaPage);
        mbar_wait(&sfull[s], (g >> 1) & 1);
        if (threadIdx.x == 0) mla_trace(3, g);  // 3: S ready at the softmax warps
        tc_fence_after();
        uint32_t sv[C::kSAcc][HG];
#pragma unroll
        for (int j = 0; j < C::kSAcc; ++j) tmem_ld8(trow + C::kSCol + (s * C::kSAcc + j) * 16 + col0, sv[j]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[s]);
        // M = 64 accumulator: token 16*q + lane sits in TMEM lane 32*q + lane (lanes < 16)
        const int tok = q * 16 + lane;
        const bool valid = lane < 16 && tok < n;
        float x[HG];
        bool over = false;
#pragma unroll
        for (int h = 0; h < HG; ++h) {
          float acc = __uint_as_float(sv[0][h]);
#pragma unroll
          for (int j = 1; j < C::kSAcc; ++j) acc += __uint_as_float(sv[j][h]);
          x[h] = valid ? acc * scale_log2 : -INFINITY;
          over |= x[h] > m_used[h] + (float)MGB_MLA_SLACK;  // (m_used = -inf: every valid score)
        }
        float alpha[HG];
        bool rescale = false;  // group-uniform (every thread derives it from the same gred values)
        if (grp_bar_or(grp, over)) {  // slow path: exchange the page maxima
          float r[HG];
#pragma unroll
          for (int h = 0; h < HG; ++h) r[h] = x[h];
          const float wmax = xreduce8<true>(r, lane);  // lane l (< 16, even) holds head (l >> 1) & 7
          if (lane < 16 && !(lane & 1)) gred[(s * 4 + q) * 16 + col0 + (lane >> 1)] = wmax;
          grp_bar(grp);
#pragma unroll
          for (int h = 0; h < HG; ++h) {
            const float* rr = gred + s * 64 + col0 + h;
            const float pm = fmaxf(fmaxf(rr[0], rr[16]), fmaxf(rr[32], rr[48]));
            alpha[h] = 1.f;
            if (pm > m_used[h] + 8.f) {
              alpha[h] = exp2f(m_used[h] - pm);  // 0 on the first page (m_used = -inf)
              m_used[h] = pm;
              rescale = true;
            }
          }
        }
        if (rescale) {
#pragma unroll
          for (int h = 0; h < HG; ++h) lpart[h] *= alpha[h];
          if (p > 0) {  // O holds pages 0..p-1: wait for the last of them, then scale it in TMEM
            wait_pv_upto(g - 1);
            tc_fence_after();
            uint32_t v[C::MT][HG];
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt) tmem_ld8(trow + ocol + mt * 16, v[mt]);
            tmem_ld_wait();
#pragma unroll
            for (int mt = 0; mt < C::MT; ++mt) {
#pragma unroll
              for (int h = 0; h < HG; ++h) v[mt][h] = __float_as_uint(__uint_as_float(v[mt][h]) * alpha[h]);
              tmem_st8(trow + ocol + mt * 16, v[mt]);
            }
            tmem_st_wait();
          }
        }
        float pv[HG];
#pragma unroll
        for (int h = 0; h < HG; ++h) {
          pv[h] = exp2f(x[h] - m_used[h]);
          lpart[h] += pv[h];
        }
        if (lane < 16) {  // P^T layout [2 head groups][64 tok][8 heads]
          uint8_t* pd = p_s + s * C::kPBytes + (grp * kMlaTile + tok) * 16;
          *reinterpret_cast<uint4*>(pd) = make_uint4(pack_bf16x2(pv[0], pv[1]), pack_bf16x2(pv[2], pv[3]),
                                                     pack_bf16x2(pv[4], pv[5]), pack_bf16x2(pv[6], pv[7]));
        }
        if (n < kMlaPage) {  // rows past the sequence end: P = 0, and V must not hold NaN/Inf
          const int tail = kMlaPage - n;
          uint8_t* pg = pages + st * C::kPageBytes + n * 128;  // token rows are contiguous 128 B
          for (int i = threadIdx.x; i < tail * 8 * C::NKB; i += 256) {  // (P.V's phantom rows alias the next block)
            const int kb = i / (tail * 8), rr = i - kb * tail * 8;
            *reinterpret_cast<uint4*>(pg + kb * C::kBlockBytes + rr * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();  // the O rescale's TMEM stores precede the next P.V (ordered by pfull)
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[s]);
        if (threadIdx.x == 0) mla_trace(4, g);    // 4: P written (warp 0, heads 0-7)
        if (threadIdx.x == 128) mla_trace(6, g);  // 6: P written (warp 4, heads 8-15)
        wait_pv_upto(g - 1);  // keep pace with the P.V stream (see wait_pv_upto)
      }
      // ---- the item's O: wait for its last P.V, normalise, store; free the O buffer ----
      wait_pv_upto(g - 1);
      tc_fence_after();
      uint32_t ov[C::MT][HG];
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) tmem_ld8(trow + ocol + mt * 16, ov[mt]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&oempty[ob]);
      ++items_sm;
      if (threadIdx.x == 0) mla_trace(9, g - 1);  // 9: item's O pulled

      // ---- normalise and store: lane = latent dim, the group's 8 heads per thread ----
      const float lsum = xreduce8<false>(lpart, lane);
      if (lane < 16 && !(lane & 1)) lred[q * 16 + col0 + (lane >> 1)] = lsum;
      grp_bar(grp);
      float inv[HG];
#pragma unroll
      for (int h = 0; h < HG; ++h) {
        const int c = col0 + h;
        const float l = lred[c] + lred[16 + c] + lred[32 + c] + lred[48 + c];
        inv[h] = l > 0.f ? __fdividef(1.0f, l) : 0.f;  // approximate: far below bf16 rounding
      }
#pragma unroll
      for (int h = 0; h < HG; ++h) {
        const int hh = hg * kMlaHeads + col0 + h;
        if (hh < H) {
          __nv_bfloat16* dst = o_lat + ((size_t)hh * B + b) * R + q * 32 + lane;
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) dst[mt * 128] = __float2bfloat16_rn(__uint_as_float(ov[mt][h]) * inv[h]);
        }
      }
      if (threadIdx.x == 0) mla_trace(10, g - 1);  // 10: O stores issued
      grp_bar(grp);  // lred reused by the next item
    }
  }
  tc_fence_before();
  __syncthreads();
  if (cl > 1) cluster_sync();  // no CTA leaves while a peer may still multicast into it / arrive on it
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

template <int R, int RP>
int launch_mla(const void* q_lat, const void* q_pe, const void* cache, const int* bt, int max_pages, const int* lens,
               int B, int H, float scale, void* out, cudaStream_t st) {
  using C = MlaCfg<R, RP>;
  if (const int rc = mgb_host::ensure_max_smem((const void*)decode_attn_mla_kernel<R, RP>, (int)C::kSmem)) return rc;
  const int n_hg = (H + kMlaHeads - 1) / kMlaHeads;
  const int items = B * n_hg;
  // the head groups of a sequence share its latent pages.  Default: independent CTAs on neighbouring
  // SMs, the pages shared through L2 (consecutive items are the head groups of one sequence, so each
  // page is read from HBM about once).  MGB_MLA_CLUSTER=1: one cluster per sequence whose leader
  // multicasts each page into all of its CTAs (L2 -> SM traffic once per sequence as well) --
  // measured slower at 128 heads (1.43 vs 1.04 ms, B=1024, ctx 640): the kernel is bound by the
  // per-page chain of each head group, and the cluster makes its CTAs wait for the slowest one.
  static const bool cl_env = [] {
    const char* e = getenv("MGB_MLA_CLUSTER");
    return e && e[0] == '1';
  }();
  const int cl = (cl_env && (n_hg == 2 || n_hg == 4 || n_hg == 8)) ? n_hg : 1;
  int grid = mgb_host::num_sms();
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  if (cl > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(kMlaThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.gridDim = dim3(grid / cl * cl);
    int nclusters = 0;  // co-resident clusters: the persistent grid must fit in one wave
    if (cudaOccupancyMaxActiveClusters(&nclusters, decode_attn_mla_kernel<R, RP>, &cfg) != cudaSuccess ||
        nclusters < 1)
      return mgb_host::launch_status(), MGB_ECUDA;
    grid = std::min(nclusters * cl, grid / cl * cl);
  }
  if (grid > items) grid = (items + cl - 1) / cl * cl;
  static const int pf_dist = [] {
    const char* e = getenv("MGB_MLA_PREFETCH");
    return e ? atoi(e) : 4;
  }();
  // Q operands straight from q_lat [H,B,R] / q_pe [B,H,RP] into the swizzled K-major
  // [block][head][64 dims] layout.  q_lat: dim0 = 64 dims of a block, dim1 = head, dim2 = block,
  // dim3 = sequence (one TMA for all R/64 blocks); q_pe: dims, head, sequence (one per block).
  CUtensorMap tq, tp;
  {
    const uint64_t d[4] = {64, (uint64_t)H, R / 64, (uint64_t)B};
    const uint64_t s[3] = {(uint64_t)B * R * 2, 128, (uint64_t)R * 2};
    const uint32_t box[4] = {64, kMlaHeads, R / 64, 1};
    if (mgb_host::encode_tmap_bf16(&tq, q_lat, 4, d, s, box, true) != CUDA_SUCCESS) return MGB_ECUDA;
  }
  {
    const uint64_t d[3] = {RP, (uint64_t)H, (uint64_t)B};
    const uint64_t s[2] = {(uint64_t)RP * 2, (uint64_t)H * RP * 2};
    const uint32_t box[3] = {64, kMlaHeads, 1};
    if (mgb_host::encode_tmap_bf16(&tp, q_pe, 3, d, s, box, true) != CUDA_SUCCESS) return MGB_ECUDA;
  }
  if (cl > 1) {
    cfg.gridDim = dim3(grid);
    cfg.stream = st;
    const __nv_bfloat16* cp = reinterpret_cast<const __nv_bfloat16*>(cache);
    __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(out);
    const float sl2 = scale * 1.4426950408889634f;
    mgb_host::launch(decode_attn_mla_kernel<R, RP>, dim3(grid), dim3(kMlaThreads), C::kSmem, st, &attr[0], tq, tp,
                     cp, bt, max_pages, lens, B, H, sl2, op, pf_dist, cl);
    return mgb_host::launch_status();
  }
  mgb_host::launch(decode_attn_mla_kernel<R, RP>, dim3(grid), dim3(kMlaThreads), C::kSmem, st, nullptr,
      tq, tp, reinterpret_cast<const __nv_bfloat16*>(cache), bt, max_pages, lens, B, H, scale * 1.4426950408889634f,
      reinterpret_cast<__nv_bfloat16*>(out), pf_dist, 1);
  return mgb_host::launch_status();
}

// Per token: latent RMSNorm (kv_a_layernorm) + interleaved RoPE of the shared k_pe, appended to
// the latent page; q_pe rotated into [B, H, RP]; q_nope rearranged into [H, B, NOPE] for the
// absorption bmm.  RoPE = HF apply_rotary_emb (fp32 complex rotation, one bf16 cast).
__global__ void mla_append_kernel(const __nv_bfloat16* __restrict__ q,    // [B, H, NOPE + RP]
                                  const __nv_bfloat16* __restrict__ ckv,  // [B, R + RP]
                                  const __nv_bfloat16* __restrict__ norm_w, float eps, int B, int H, int R, int RP,
                                  int NOPE, const int* __restrict__ positions, const float* __restrict__ cos_t,
                                  const float* __restrict__ sin_t, const int* __restrict__ block_table, int max_pages,
                                  __nv_bfloat16* __restrict__ cache, __nv_bfloat16* __restrict__ q_nope_out,
                                  __nv_bfloat16* __restrict__ q_pe_out, int* __restrict__ seq_lens) {
  mgb::pdl_enter();
  const int b = blockIdx.x;
  const int pos = positions[b];
  if (pos < 0 || pos >= max_pages * kMlaPage) return;  // past the planned context: no page to write
  const int D = R + RP;
  __shared__ float red[32];
  const __nv_bfloat16* row = ckv + (size_t)b * D;
  const int page = block_table[(size_t)b * max_pages + pos / kMlaPage];
  const int slot = pos % kMlaPage;
  const int DP = (D + 63) / 64 * 64;  // padded page row (see the page layout above)
  __nv_bfloat16* pg = cache + (size_t)page * DP * kMlaPage;
  // element offset of dim i of this token inside the swizzled page
  auto at = [slot](int i) { return (i >> 6) * (kMlaPage * 64) + slot * 64 + ((((i >> 3) & 7) ^ (slot & 7)) << 3) + (i & 7); };
  if (seq_lens && threadIdx.x == 0) seq_lens[b] = pos + 1;
  // latent RMSNorm (HF DeepseekV2RMSNorm: fp32 variance, bf16 cast, times weight)
  float ss = 0.f;
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const float v = __bfloat162float(row[i]);
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += red[i];
  const float inv = 1.0f / sqrtf(tot / (float)R + eps);
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const float v = __bfloat162float(norm_w[i]) * bf16_round(__bfloat162float(row[i]) * inv);
    pg[at(i)] = __float2bfloat16_rn(v);
  }
  const float* cs = cos_t + (size_t)pos * (RP / 2);
  const float* sn = sin_t + (size_t)pos * (RP / 2);
  for (int i = threadIdx.x; i < RP / 2; i += blockDim.x) {  // shared k_pe
    const float x0 = __bfloat162float(row[R + 2 * i]), x1 = __bfloat162float(row[R + 2 * i + 1]);
    const float c = cs[i], s = sn[i];
    const int d0 = R + 2 * i;
    pg[at(d0)] = __float2bfloat16_rn(x0 * c - x1 * s);
    pg[at(d0 + 1)] = __float2bfloat16_rn(x0 * s + x1 * c);
  }
  // the row's padding dims [D, DP) must be finite whatever the page held before: P.V's phantom rows
  // read them (times P = 0) for the page's first 8 tokens, and 0 * NaN would poison O
  for (int i = D + threadIdx.x; i < DP; i += blockDim.x) pg[at(i)] = __float2bfloat16_rn(0.f);
  const int QD = NOPE + RP;
  for (int i = threadIdx.x; i < H * (RP / 2); i += blockDim.x) {  // per-head q_pe
    const int h = i / (RP / 2), j = i - h * (RP / 2);
    const __nv_bfloat16* qh = q + ((size_t)b * H + h) * QD + NOPE;
    const float x0 = __bfloat162float(qh[2 * j]), x1 = __bfloat162float(qh[2 * j + 1]);
    const float c = cs[j], s = sn[j];
    __nv_bfloat16* dst = q_pe_out + ((size_t)b * H + h) * RP + 2 * j;
    dst[0] = __float2bfloat16_rn(x0 * c - x1 * s);
    dst[1] = __float2bfloat16_rn(x0 * s + x1 * c);
  }
  for (int i = threadIdx.x; i < H * (NOPE / 8); i += blockDim.x) {  // q_nope -> [H, B, NOPE]
    const int h = i / (NOPE / 8), c = i - h * (NOPE / 8);
    *reinterpret_cast<uint4*>(q_nope_out + ((size_t)h * B + b) * NOPE + c * 8) =
        *reinterpret_cast<const uint4*>(q + ((size_t)b * H + h) * QD + c * 8);
  }
}

// Warp-per-token version of mla_append_kernel (same arithmetic; the variance is summed per lane then
// across the warp): 16-byte loads and stores throughout, every load of a token's latent row and of a
// batch of its q row in flight together, 8 tokens per CTA -- the decode step's append was a chain of
// scalar loads / block barriers per token (DSV2-Lite B = 6058: 41 us per layer).
constexpr int kAppTok = 8;  // tokens (warps) per CTA
MGB_DEVINL uint4 rope_pairs(uint4 v, const float* cs, const float* sn, int pair0) {
  // interleaved RoPE on the 4 (even, odd) pairs of one 16-byte chunk; fp32 rotation, one bf16 cast
  float x[8] = {bf16lo(v.x), bf16hi(v.x), bf16lo(v.y), bf16hi(v.y), bf16lo(v.z), bf16hi(v.z), bf16lo(v.w), bf16hi(v.w)};
  float y[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float c = cs[pair0 + i], s = sn[pair0 + i];
    y[2 * i] = x[2 * i] * c - x[2 * i + 1] * s;
    y[2 * i + 1] = x[2 * i] * s + x[2 * i + 1] * c;
  }
  return make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]), pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
}

__global__ void __launch_bounds__(kAppTok * 32)
mla_append_warp_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ ckv,
                       const __nv_bfloat16* __restrict__ norm_w, float eps, int B, int H, int R, int RP, int NOPE,
                       const int* __restrict__ positions, const float* __restrict__ cos_t,
                       const float* __restrict__ sin_t, const int* __restrict__ block_table, int max_pages,
                       __nv_bfloat16* __restrict__ cache, __nv_bfloat16* __restrict__ q_nope_out,
                       __nv_bfloat16* __restrict__ q_pe_out, int* __restrict__ seq_lens) {
  mgb::pdl_enter();
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * kAppTok + (threadIdx.x >> 5);
  if (b >= B) return;
  const int pos = positions[b];
  if (pos < 0 || pos >= max_pages * kMlaPage) return;  // past the planned context: no page to write
  const int D = R + RP, DP = (D + 63) / 64 * 64;
  const int nR = R / 8, nD = D / 8, nDP = DP / 8;     // 16-byte chunks: latent, row, padded row
  constexpr int kLat = 4;                              // latent-row chunks per lane (D <= 1024)
  const uint4* row = reinterpret_cast<const uint4*>(ckv + (size_t)b * D);
  uint4 v[kLat];
#pragma unroll
  for (int u = 0; u < kLat; ++u)
    if (lane + 32 * u < nD) v[u] = ld_nc_v4(row + lane + 32 * u);
  const int page = block_table[(size_t)b * max_pages + pos / kMlaPage];
  const int slot = pos % kMlaPage;
  uint4* pg = reinterpret_cast<uint4*>(cache + (size_t)page * DP * kMlaPage);
  // chunk c (8 dims) of this token inside the swizzled page: block c / 8, row `slot`, chunk c ^ slot
  auto at = [slot](int c) { return (c >> 3) * (kMlaPage * 8) + slot * 8 + ((c & 7) ^ (slot & 7)); };
  if (seq_lens && lane == 0) seq_lens[b] = pos + 1;
  const float* cs = cos_t + (size_t)pos * (RP / 2);
  const float* sn = sin_t + (size_t)pos * (RP / 2);
  // latent RMSNorm (HF DeepseekV2RMSNorm: fp32 variance, bf16 cast, times weight)
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < kLat; ++u) {
    const int c = lane + 32 * u;
    if (c < nR) {
      const float f[8] = {bf16lo(v[u].x), bf16hi(v[u].x), bf16lo(v[u].y), bf16hi(v[u].y),
                          bf16lo(v[u].z), bf16hi(v[u].z), bf16lo(v[u].w), bf16hi(v[u].w)};
#pragma unroll
      for (int i = 0; i < 8; ++i) ss = fmaf(f[i], f[i], ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = 1.0f / sqrtf(ss / (float)R + eps);
#pragma unroll
  for (int u = 0; u < kLat; ++u) {
    const int c = lane + 32 * u;
    if (c < nR) {
      const uint4 w = ld_nc_v4(reinterpret_cast<const uint4*>(norm_w) + c);
      const float f[8] = {bf16lo(v[u].x), bf16hi(v[u].x), bf16lo(v[u].y), bf16hi(v[u].y),
                          bf16lo(v[u].z), bf16hi(v[u].z), bf16lo(v[u].w), bf16hi(v[u].w)};
      const float wf[8] = {bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y), bf16lo(w.z), bf16hi(w.z), bf16lo(w.w), bf16hi(w.w)};
      float y[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) y[i] = wf[i] * bf16_round(f[i] * inv);
      pg[at(c)] = make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]), pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
    } else if (c < nD) {  // the shared k_pe: interleaved RoPE
      pg[at(c)] = rope_pairs(v[u], cs, sn, (c - nR) * 4);
    } else if (c < nDP) {  // padding dims: finite (P.V's phantom rows read them times P = 0)
      pg[at(c)] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  // q row [H, NOPE + RP]: q_nope -> [H, B, NOPE], q_pe RoPE'd -> [B, H, RP]; kQ chunks per lane in flight
  const int qc = (NOPE + RP) / 8, nq = H * qc, nope_c = NOPE / 8;
  const uint4* qrow = reinterpret_cast<const uint4*>(q + (size_t)b * H * (NOPE + RP));
  constexpr int kQ = 8;
  for (int c0 = lane; c0 < nq; c0 += 32 * kQ) {
    uint4 x[kQ];
#pragma unroll
    for (int u = 0; u < kQ; ++u)
      if (c0 + 32 * u < nq) x[u] = ld_nc_v4(qrow + c0 + 32 * u);
#pragma unroll
    for (int u = 0; u < kQ; ++u) {
      const int c = c0 + 32 * u;
      if (c >= nq) continue;
      const int h = c / qc, cc = c - h * qc;
      if (cc < nope_c)
        reinterpret_cast<uint4*>(q_nope_out + ((size_t)h * B + b) * NOPE)[cc] = x[u];
      else
        reinterpret_cast<uint4*>(q_pe_out + ((size_t)b * H + h) * RP)[cc - nope_c] = rope_pairs(x[u], cs, sn, (cc - nope_c) * 4);
    }
  }
}

// Prefill variant (T = n_seq * P prompt tokens; token t = position t % P of sequence seq0 + t / P):
// the normed latent + RoPE'd k_pe of every prompt token into the latent pages, and contiguous copies
// for the (non-absorbed) causal prefill attention: c_out [T, R], kpe_out [T, RP]; the q_pe part of
// each row of q [T, H, NOPE + RP] is rotated in place.  Same arithmetic as mla_append_kernel.
__global__ void mla_append_prefill_kernel(__nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ ckv,
                                          const __nv_bfloat16* __restrict__ norm_w, float eps, int seq0, int P, int H,
                                          int R, int RP, int NOPE, const float* __restrict__ cos_t,
                                          const float* __restrict__ sin_t, const int* __restrict__ block_table,
                                          int max_pages, __nv_bfloat16* __restrict__ cache,
                                          __nv_bfloat16* __restrict__ c_out, __nv_bfloat16* __restrict__ kpe_out) {
  mgb::pdl_enter();
  const int t = blockIdx.x;
  const int seq = seq0 + t / P, pos = t % P;
  const int D = R + RP;
  __shared__ float red[32];
  const __nv_bfloat16* row = ckv + (size_t)t * D;
  const int page = block_table[(size_t)seq * max_pages + pos / kMlaPage];
  const int slot = pos % kMlaPage;
  const int DP = (D + 63) / 64 * 64;
  __nv_bfloat16* pg = cache + (size_t)page * DP * kMlaPage;
  auto at = [slot](int i) { return (i >> 6) * (kMlaPage * 64) + slot * 64 + ((((i >> 3) & 7) ^ (slot & 7)) << 3) + (i & 7); };
  float ss = 0.f;
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const float v = __bfloat162float(row[i]);
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += red[i];
  const float inv = 1.0f / sqrtf(tot / (float)R + eps);
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    const __nv_bfloat16 v = __float2bfloat16_rn(__bfloat162float(norm_w[i]) * bf16_round(__bfloat162float(row[i]) * inv));
    pg[at(i)] = v;
    c_out[(size_t)t * R + i] = v;
  }
  const float* cs = cos_t + (size_t)pos * (RP / 2);
  const float* sn = sin_t + (size_t)pos * (RP / 2);
  for (int i = threadIdx.x; i < RP / 2; i += blockDim.x) {  // shared k_pe
    const float x0 = __bfloat162float(row[R + 2 * i]), x1 = __bfloat162float(row[R + 2 * i + 1]);
    const float c = cs[i], s = sn[i];
    const __nv_bfloat16 a = __float2bfloat16_rn(x0 * c - x1 * s), b = __float2bfloat16_rn(x0 * s + x1 * c);
    pg[at(R + 2 * i)] = a;
    pg[at(R + 2 * i + 1)] = b;
    kpe_out[(size_t)t * RP + 2 * i] = a;
    kpe_out[(size_t)t * RP + 2 * i + 1] = b;
  }
  for (int i = D + threadIdx.x; i < DP; i += blockDim.x) pg[at(i)] = __float2bfloat16_rn(0.f);  // padding
  const int QD = NOPE + RP;
  for (int i = threadIdx.x; i < H * (RP / 2); i += blockDim.x) {  // per-head q_pe, in place
    const int h = i / (RP / 2), j = i - h * (RP / 2);
    __nv_bfloat16* qh = q + ((size_t)t * H + h) * QD + NOPE;
    const float x0 = __bfloat162float(qh[2 * j]), x1 = __bfloat162float(qh[2 * j + 1]);
    const float c = cs[j], s = sn[j];
    qh[2 * j] = __float2bfloat16_rn(x0 * c - x1 * s);
    qh[2 * j + 1] = __float2bfloat16_rn(x0 * s + x1 * c);
  }
}

}  // namespace mgb

extern "C" {

int mgb_mla_page_size(void) { return mgb::kMlaPage; }

// bf16 elements of one latent page for latent width R and rope width RP (rows padded to 64).
int mgb_mla_page_elems(int R, int RP) { return (R + RP + 63) / 64 * 64 * mgb::kMlaPage; }

// Absorbed MLA decode attention: q_lat [H,B,R], q_pe [B,H,RP], latent pages -> o_lat [H,B,R].
int mgb_decode_attn_mla(const void* q_lat, const void* q_pe, const void* cache, const int* block_table, int max_pages,
                        const int* seq_lens, int B, int H, int R, int RP, float scale, void* o_lat, void* stream) {
  if (B < 1 || H < 1) return MGB_EINVAL;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (R == 512 && RP == 64) return mgb::launch_mla<512, 64>(q_lat, q_pe, cache, block_table, max_pages, seq_lens, B, H, scale, o_lat, st);
  if (R == 128 && RP == 32) return mgb::launch_mla<128, 32>(q_lat, q_pe, cache, block_table, max_pages, seq_lens, B, H, scale, o_lat, st);
  return MGB_EINVAL;
}

// Latent KV append (+ q_pe RoPE and q_nope re-layout) for one new token per sequence.
int mgb_mla_append(const void* q, const void* ckv, const void* norm_w, float eps, int B, int H, int R, int RP, int NOPE,
                   const int* positions, const float* cos_t, const float* sin_t, const int* block_table, int max_pages,
                   void* cache, void* q_nope_out, void* q_pe_out, int* seq_lens, void* stream) {
  if (B < 1 || H < 1 || R % 8 || RP % 8 || NOPE % 8) return MGB_EINVAL;
  const char* blk = getenv("MGB_MLA_APPEND_BLOCK");  // the per-token-CTA kernel (A/B and tests)
  if (!(blk && blk[0] == '1') && ((R + RP + 63) / 64 * 64) <= 1024) {
    mgb_host::launch(mgb::mla_append_warp_kernel, dim3((B + mgb::kAppTok - 1) / mgb::kAppTok), dim3(mgb::kAppTok * 32), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
        reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(ckv),
        reinterpret_cast<const __nv_bfloat16*>(norm_w), eps, B, H, R, RP, NOPE, positions, cos_t, sin_t, block_table,
        max_pages, reinterpret_cast<__nv_bfloat16*>(cache), reinterpret_cast<__nv_bfloat16*>(q_nope_out),
        reinterpret_cast<__nv_bfloat16*>(q_pe_out), seq_lens);
    return mgb_host::launch_status();
  }
  mgb_host::launch(mgb::mla_append_kernel, dim3(B), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(ckv),
      reinterpret_cast<const __nv_bfloat16*>(norm_w), eps, B, H, R, RP, NOPE, positions, cos_t, sin_t, block_table,
      max_pages, reinterpret_cast<__nv_bfloat16*>(cache), reinterpret_cast<__nv_bfloat16*>(q_nope_out),
      reinterpret_cast<__nv_bfloat16*>(q_pe_out), seq_lens);
  return mgb_host::launch_status();
}

// Prefill: latent + k_pe of T = n_seq * P prompt tokens into the pages and contiguous rows; q_pe RoPE
// in place.
int mgb_mla_append_prefill(void* q, const void* ckv, const void* norm_w, float eps, int T, int seq0, int P, int H,
                           int R, int RP, int NOPE, const float* cos_t, const float* sin_t, const int* block_table,
                           int max_pages, void* cache, void* c_out, void* kpe_out, void* stream) {
  if (T < 1 || P < 1 || T % P || H < 1 || R % 8 || RP % 8 || NOPE % 8) return MGB_EINVAL;
  mgb_host::launch(mgb::mla_append_prefill_kernel, dim3(T), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), nullptr,
      reinterpret_cast<__nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(ckv),
      reinterpret_cast<const __nv_bfloat16*>(norm_w), eps, seq0, P, H, R, RP, NOPE, cos_t, sin_t, block_table, max_pages,
      reinterpret_cast<__nv_bfloat16*>(cache), reinterpret_cast<__nv_bfloat16*>(c_out),
      reinterpret_cast<__nv_bfloat16*>(kpe_out));
  return mgb_host::launch_status();
}

#ifdef MGB_MLA_TRACE
int mgb_mla_trace_read(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, mgb::g_mla_trace, sizeof(mgb::g_mla_trace)) == cudaSuccess ? MGB_OK : MGB_ECUDA;
}
#endif

}  // extern "C"
