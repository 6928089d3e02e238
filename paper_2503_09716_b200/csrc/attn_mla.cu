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
// Latent cache: pages of kMlaPage = 32 tokens, chunk-major [(R+r)/8][32 tok][8] bf16, so every
// ldmatrix / ldmatrix.trans is conflict free and a page is one contiguous bulk copy.
// Persistent kernel, 2 CTAs per SM: warp 4 streams pages through a 2-stage ring
// (cp.async.bulk + mbarrier); warps 0-3 consume.  Per page: each warp computes S = Q C^T for 8
// tokens x 16 heads on the tensor cores (Q in padded smem, ldmatrix A fragments), the four warps
// run one online-softmax pass over the 32 tokens in smem, then each warp accumulates O for its
// quarter of the latent dims with P V on the tensor cores.  A work item is (sequence, 16-head group).
#include "common.cuh"

namespace mgb {

constexpr int kMlaPage = 32;
constexpr int kMlaStages = 2;
constexpr int kMlaConsumers = 4;
constexpr int kMlaThreads = (kMlaConsumers + 1) * 32;

MGB_DEVINL void ldsm4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
MGB_DEVINL void ldsm4t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
MGB_DEVINL void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
MGB_DEVINL void cons_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <int R, int RP>  // latent width, rope width
struct MlaCfg {
  static constexpr int D = R + RP;                     // cached row width
  static constexpr int NCH = D / 8;                    // 16 B chunks per row
  static constexpr int kPageBytes = D * kMlaPage * 2;  // one page, contiguous
  static constexpr int kQStride = D * 2 + 16;          // padded smem row (bytes) -> conflict-free ldmatrix
  static constexpr int kPStride = kMlaPage * 2 + 16;   // padded P row (bytes)
  static constexpr int DPW = R / kMlaConsumers;         // latent dims of O per warp
  static constexpr int NT = DPW / 8;                    // PV n-tiles per warp
  static constexpr int KST = D / 16;                   // k-steps of S = Q C^T
  static constexpr int KPW = (KST + kMlaConsumers - 1) / kMlaConsumers;  // k-steps per warp (K split)
  static constexpr size_t kSmem = (size_t)kMlaStages * kPageBytes + 16 * kQStride +
                                  kMlaConsumers * 16 * kMlaPage * 4 + 2 * 16 * kPStride + 16 * 4 * 4 + 64;
  static_assert(R % (8 * kMlaConsumers * 2) == 0 && D % 32 == 0, "MLA shape");
};

template <int R, int RP>
__global__ void __launch_bounds__(kMlaThreads, 2)
decode_attn_mla_kernel(const __nv_bfloat16* __restrict__ q_lat,  // [H, B, R]
                       const __nv_bfloat16* __restrict__ q_pe,   // [B, H, RP]
                       const __nv_bfloat16* __restrict__ cache,  // latent pages
                       const int* __restrict__ block_table, int max_pages, const int* __restrict__ seq_lens,
                       int B, int H, float scale_log2, __nv_bfloat16* __restrict__ o_lat) {  // [H, B, R]
  using C = MlaCfg<R, RP>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint8_t* q_s = smem + kMlaStages * C::kPageBytes;                                   // [16][kQStride]
  float* s_s = reinterpret_cast<float*>(q_s + 16 * C::kQStride);                      // [warp][16][32] partial S
  uint8_t* p_s = reinterpret_cast<uint8_t*>(s_s + kMlaConsumers * 16 * kMlaPage);     // [2][16][kPStride]
  float* m_s = reinterpret_cast<float*>(p_s + 2 * 16 * C::kPStride);                 // [16]
  float* l_s = m_s + 16;
  float* a_s = l_s + 16;                                                               // alpha [16]
  uint64_t* full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(a_s + 32) + 15) & ~uintptr_t(15));
  uint64_t* empty = full + kMlaStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_hg = (H + 15) / 16;
  const int n_items = B * n_hg;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMlaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kMlaConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kMlaConsumers) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int b = it / n_hg;
        const int np = (seq_lens[b] + kMlaPage - 1) / kMlaPage;
        const int* bt = block_table + (size_t)b * max_pages;
        for (int p = 0; p < np; ++p) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::kPageBytes);
          bulk_load(ring + stage * C::kPageBytes, cache + (size_t)bt[p] * (C::kPageBytes / 2), C::kPageBytes,
                    &full[stage], pol);
          if (++stage == kMlaStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  const int g = lane >> 2, t = lane & 3;
  const int tid = threadIdx.x;  // 0..127
  int stage = 0;
  uint32_t phase = 0;
  int sbuf = 0;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int b = it / n_hg, hg = it - b * n_hg;
    const int len = seq_lens[b];
    const int np = (len + kMlaPage - 1) / kMlaPage;
    // ---- stage Q = [q_lat | q_pe] for the 16 heads of the group (rows >= H are zero) ----
    for (int i = tid; i < 16 * C::NCH; i += 128) {
      const int row = i / C::NCH, ch = i - row * C::NCH;
      const int h = hg * 16 + row;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (h < H) {
        v = ch < R / 8 ? *reinterpret_cast<const uint4*>(q_lat + ((size_t)h * B + b) * R + ch * 8)
                       : *reinterpret_cast<const uint4*>(q_pe + ((size_t)b * H + h) * RP + (ch - R / 8) * 8);
      }
      *reinterpret_cast<uint4*>(q_s + row * C::kQStride + ch * 16) = v;
    }
    if (tid < 16) {
      m_s[tid] = -INFINITY;
      l_s[tid] = 0.f;
    }
    float o[C::NT][4];
#pragma unroll
    for (int n = 0; n < C::NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    cons_bar();

    const uint32_t qbase = smem_u32(q_s);
    // this warp's K-split share of Q (k-steps warp, warp+4, ...) lives in registers for the item
    uint32_t qa[C::KPW][4];
    {
      const int mi = lane >> 3, r = lane & 7;
#pragma unroll
      for (int kk = 0; kk < C::KPW; ++kk) {
        const int ks = warp + kMlaConsumers * kk;
        if (ks < C::KST)
          ldsm4(qbase + (uint32_t)(((mi & 1) * 8 + r) * C::kQStride + (ks * 16 + (mi >> 1) * 8) * 2), qa[kk][0],
                qa[kk][1], qa[kk][2], qa[kk][3]);
      }
    }
    for (int p = 0; p < np; ++p) {
      mbar_wait(&full[stage], phase);
      const uint32_t cbase = smem_u32(ring + stage * C::kPageBytes);
      float* S = s_s;
      uint8_t* P = p_s + sbuf * 16 * C::kPStride;
      // ---- partial S[16 x 32] over this warp's k-steps (4 independent n-tile accumulators) ----
      {
        float acc[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        const int mi = lane >> 3, r = lane & 7;
#pragma unroll
        for (int kk = 0; kk < C::KPW; ++kk) {
          const int ks = warp + kMlaConsumers * kk;
          if (ks < C::KST) {
            // matrices (chunk 2ks, tok 0-7), (chunk 2ks+1, tok 0-7), (chunk 2ks, tok 8-15), (chunk 2ks+1, tok 8-15)
            uint32_t b0, b1, b2, b3, b4, b5, b6, b7;
            const uint32_t kaddr = cbase + (uint32_t)(((2 * ks + (mi & 1)) * kMlaPage + (mi >> 1) * 8 + r) * 16);
            ldsm4(kaddr, b0, b1, b2, b3);
            ldsm4(kaddr + 16 * 16, b4, b5, b6, b7);  // tokens 16..31
            mma16816(acc[0], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
            mma16816(acc[1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b2, b3);
            mma16816(acc[2], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b4, b5);
            mma16816(acc[3], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b6, b7);
          }
        }
        float* Sw = S + warp * 16 * kMlaPage;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = j * 8 + 2 * t;
          *reinterpret_cast<float2*>(Sw + g * kMlaPage + col) = make_float2(acc[j][0], acc[j][1]);
          *reinterpret_cast<float2*>(Sw + (g + 8) * kMlaPage + col) = make_float2(acc[j][2], acc[j][3]);
        }
      }
      cons_bar();
      // ---- online softmax: warp w owns rows 4w..4w+3, lane = token ----
      {
        const int n = min(kMlaPage, len - p * kMlaPage);
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const int row = warp * 4 + rr;
          float sv = -INFINITY;
          if (lane < n) {
            sv = 0.f;
#pragma unroll
            for (int w = 0; w < kMlaConsumers; ++w) sv += S[(w * 16 + row) * kMlaPage + lane];
            sv *= scale_log2;
          }
          float mt = sv;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
          const float m_old = m_s[row];
          const float m_new = fmaxf(m_old, mt);
          const float pv = exp2f(sv - m_new);
          float ps = pv;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
          reinterpret_cast<__nv_bfloat16*>(P + row * C::kPStride)[lane] = __float2bfloat16_rn(pv);
          __syncwarp();
          if (lane == 0) {
            const float alpha = exp2f(m_old - m_new);
            a_s[row] = alpha;
            l_s[row] = l_s[row] * alpha + ps;
            m_s[row] = m_new;
          }
        }
      }
      cons_bar();
      // ---- O[16 x DPW] = O * alpha + P[16 x 32] C[32 x DPW] ----
      {
        const float al0 = a_s[g], al1 = a_s[g + 8];
#pragma unroll
        for (int n = 0; n < C::NT; ++n) {
          o[n][0] *= al0; o[n][1] *= al0; o[n][2] *= al1; o[n][3] *= al1;
        }
        const uint32_t pbase = smem_u32(P);
        const int mi = lane >> 3, r = lane & 7;
#pragma unroll
        for (int ks = 0; ks < kMlaPage / 16; ++ks) {
          uint32_t a0, a1, a2, a3;
          ldsm4(pbase + (uint32_t)(((mi & 1) * 8 + r) * C::kPStride + (ks * 16 + (mi >> 1) * 8) * 2), a0, a1, a2, a3);
#pragma unroll
          for (int n2 = 0; n2 < C::NT / 2; ++n2) {
            const int chunk = warp * (C::DPW / 8) + 2 * n2 + (mi >> 1);
            const int tok = ks * 16 + ((mi & 1) << 3) + r;
            uint32_t v0a, v0b, v1a, v1b;
            ldsm4t(cbase + (uint32_t)((chunk * kMlaPage + tok) * 16), v0a, v0b, v1a, v1b);
            mma16816(o[2 * n2], a0, a1, a2, a3, v0a, v0b);
            mma16816(o[2 * n2 + 1], a0, a1, a2, a3, v1a, v1b);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kMlaStages) { stage = 0; phase ^= 1; }
      sbuf ^= 1;
    }
    // ---- normalise and store this warp's dims of the heads of the group ----
    cons_bar();  // l_s final for every row
    const float l0 = l_s[g], l1 = l_s[g + 8];
    const int h0 = hg * 16 + g, h1 = h0 + 8;
#pragma unroll
    for (int n = 0; n < C::NT; ++n) {
      const int dim = warp * C::DPW + n * 8 + 2 * t;
      if (h0 < H)
        *reinterpret_cast<uint32_t*>(o_lat + ((size_t)h0 * B + b) * R + dim) =
            pack_bf16x2(l0 > 0.f ? o[n][0] / l0 : 0.f, l0 > 0.f ? o[n][1] / l0 : 0.f);
      if (h1 < H)
        *reinterpret_cast<uint32_t*>(o_lat + ((size_t)h1 * B + b) * R + dim) =
            pack_bf16x2(l1 > 0.f ? o[n][2] / l1 : 0.f, l1 > 0.f ? o[n][3] / l1 : 0.f);
    }
    cons_bar();  // q_s / m_s / l_s reused by the next item
  }
}

template <int R, int RP>
int launch_mla(const void* q_lat, const void* q_pe, const void* cache, const int* bt, int max_pages, const int* lens,
               int B, int H, float scale, void* out, cudaStream_t st) {
  using C = MlaCfg<R, RP>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(decode_attn_mla_kernel<R, RP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::kSmem) != cudaSuccess)
      return MGB_ECUDA;
    attr = true;
  }
  const int items = B * ((H + 15) / 16);
  int grid = 2 * mgb_host::num_sms();
  if (grid > items) grid = items;
  decode_attn_mla_kernel<R, RP><<<grid, kMlaThreads, C::kSmem, st>>>(
      reinterpret_cast<const __nv_bfloat16*>(q_lat), reinterpret_cast<const __nv_bfloat16*>(q_pe),
      reinterpret_cast<const __nv_bfloat16*>(cache), bt, max_pages, lens, B, H, scale * 1.4426950408889634f,
      reinterpret_cast<__nv_bfloat16*>(out));
  return cudaGetLastError() == cudaSuccess ? MGB_OK : MGB_ECUDA;
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
  const int b = blockIdx.x;
  const int pos = positions[b];
  const int D = R + RP;
  __shared__ float red[32];
  const __nv_bfloat16* row = ckv + (size_t)b * D;
  const int page = block_table[(size_t)b * max_pages + pos / kMlaPage];
  const int slot = pos % kMlaPage;
  __nv_bfloat16* pg = cache + (size_t)page * D * kMlaPage;
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
    pg[((size_t)(i / 8) * kMlaPage + slot) * 8 + (i % 8)] = __float2bfloat16_rn(v);
  }
  const float* cs = cos_t + (size_t)pos * (RP / 2);
  const float* sn = sin_t + (size_t)pos * (RP / 2);
  for (int i = threadIdx.x; i < RP / 2; i += blockDim.x) {  // shared k_pe
    const float x0 = __bfloat162float(row[R + 2 * i]), x1 = __bfloat162float(row[R + 2 * i + 1]);
    const float c = cs[i], s = sn[i];
    const int d0 = R + 2 * i;
    pg[((size_t)(d0 / 8) * kMlaPage + slot) * 8 + (d0 % 8)] = __float2bfloat16_rn(x0 * c - x1 * s);
    pg[((size_t)((d0 + 1) / 8) * kMlaPage + slot) * 8 + ((d0 + 1) % 8)] = __float2bfloat16_rn(x0 * s + x1 * c);
  }
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

}  // namespace mgb

extern "C" {

int mgb_mla_page_size(void) { return mgb::kMlaPage; }

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
  mgb::mla_append_kernel<<<B, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(ckv),
      reinterpret_cast<const __nv_bfloat16*>(norm_w), eps, B, H, R, RP, NOPE, positions, cos_t, sin_t, block_table,
      max_pages, reinterpret_cast<__nv_bfloat16*>(cache), reinterpret_cast<__nv_bfloat16*>(q_nope_out),
      reinterpret_cast<__nv_bfloat16*>(q_pe_out), seq_lens);
  return cudaGetLastError() == cudaSuccess ? MGB_OK : MGB_ECUDA;
}

}  // extern "C"
