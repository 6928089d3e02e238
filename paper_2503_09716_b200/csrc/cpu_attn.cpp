// ATTN_MECH_CPU: GQA decode attention on the host cores over the host KV page store — MoE-Gen's
// CPU attention split (omega > 0; schedule nodes offload_dag.py:328-357).
//
// The sequences [s0, s0 + B) of the plan's CPU share never have their KV copied to the GPU: their
// pages stay in pinned host memory (kv_policy "offload"), the GPU only computes their q/k/v and
// writes the new token into the host pages (KV_COPY_OUT), and the host cores run the attention
// mechanism.  In the engine this runs as a host node of the decode step's CUDA graph
// (mgb_cpu_attn_gqa_enqueue -> cudaLaunchHostFunc) between the D2H copy of q and the H2D copy of the
// output, so the CPU share overlaps the GPU's own attention micro-batches.
//
// Pages use the GPU layout (attn_gqa.cu): per (page, kv head) a block [hd/8 chunks][page tok][8].
// QK^T uses AVX-512 BF16 dot products (VDPBF16PS) on 4 tokens x 8 dims per load; PV converts V to
// fp32 and accumulates with FMAs.  Numerics: fp32 scores, fp32 softmax, probabilities rounded to
// bf16 (HF casts softmax to the value dtype, modeling_mixtral.py:285-287), fp32 PV accumulation,
// one bf16 rounding of the output.  A scalar path covers hosts without AVX-512 BF16.
#include <immintrin.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

extern "C" {
struct MgbCpuAttnGqa {
  const uint16_t* k_pages;   // host page store of the layer (bf16 bits), K
  const uint16_t* v_pages;   // V
  const uint16_t* q;         // [B, Hq, hd] bf16, RoPE applied (pinned host)
  const int32_t* seq_lens;   // [B] keys per sequence (pinned host)
  uint16_t* out;             // [B, Hq * hd] bf16 (pinned host)
  int64_t first_page;        // page of sequence 0's first token; sequence b owns pages first + b*pps ...
  int32_t pps;               // pages per sequence
  int32_t B, Hq, Hkv, hd, page_tokens;
  float scale;
  int32_t status;            // set by the callback: 0 ok, -1 invalid
};
}

namespace {

inline float bf2f(uint16_t v) {
  uint32_t u = (uint32_t)v << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
inline uint16_t f2bf(float f) {  // round to nearest even
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// ------------------------------------------------------------------------------------------
// A persistent pool of host threads (parallel_for over work items)
// ------------------------------------------------------------------------------------------
class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  void resize(int n) {
    std::lock_guard<std::mutex> g(run_mu_);
    stop_all();
    n_ = std::max(1, n);
    for (int i = 1; i < n_; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  int size() const { return n_; }
  void parallel_for(int items, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> g(run_mu_);
    if (n_ == 1 || items <= 1) {
      for (int i = 0; i < items; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> l(mu_);
      fn_ = &fn;
      items_ = items;
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(mu_);
    done_cv_.wait(l, [this] { return done_ == n_ - 1; });
    fn_ = nullptr;
  }
  ~Pool() { stop_all(); }

 private:
  Pool() {
    unsigned hc = std::thread::hardware_concurrency();
    n_ = 1;
    resize_unlocked(hc ? (int)hc : 1);
  }
  void resize_unlocked(int n) {
    n_ = std::max(1, n);
    for (int i = 1; i < n_; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  void stop_all() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
    workers_.clear();
    stop_ = false;
  }
  void work() {
    for (;;) {
      int i = next_.fetch_add(1);
      if (i >= items_) break;
      (*fn_)(i);
    }
  }
  void loop(int) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      work();
      {
        std::lock_guard<std::mutex> l(mu_);
        ++done_;
      }
      done_cv_.notify_one();
    }
  }
  int n_ = 1;
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<int> next_{0};
  int items_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// ------------------------------------------------------------------------------------------
// one (sequence, kv head): G query heads over L keys
// ------------------------------------------------------------------------------------------
constexpr int kMaxG = 16;

void softmax_round(float* s, int L, float scale) {
  float m = -INFINITY;
  for (int t = 0; t < L; ++t) m = std::max(m, s[t] * scale);
  float sum = 0.f;
  for (int t = 0; t < L; ++t) {
    s[t] = std::exp(s[t] * scale - m);
    sum += s[t];
  }
  const float inv = 1.f / sum;
  for (int t = 0; t < L; ++t) s[t] = bf2f(f2bf(s[t] * inv));  // probabilities in the value dtype
}

void head_scalar(const MgbCpuAttnGqa& d, int b, int kh, std::vector<float>& sc) {
  const int G = d.Hq / d.Hkv, hd = d.hd, P = d.page_tokens, L = d.seq_lens[b];
  const int64_t blk = (int64_t)hd * P;
  for (int g = 0; g < G; ++g) {
    const uint16_t* q = d.q + ((int64_t)b * d.Hq + kh * G + g) * hd;
    float* s = sc.data() + (int64_t)g * L;
    for (int t = 0; t < L; ++t) {
      const uint16_t* kp = d.k_pages + ((d.first_page + (int64_t)b * d.pps + t / P) * d.Hkv + kh) * blk;
      float acc = 0.f;
      for (int c = 0; c < hd / 8; ++c)
        for (int i = 0; i < 8; ++i) acc += bf2f(q[c * 8 + i]) * bf2f(kp[((int64_t)c * P + t % P) * 8 + i]);
      s[t] = acc;
    }
    softmax_round(s, L, d.scale);
    uint16_t* o = d.out + ((int64_t)b * d.Hq + kh * G + g) * hd;
    for (int c = 0; c < hd / 8; ++c)
      for (int i = 0; i < 8; ++i) {
        float acc = 0.f;
        for (int t = 0; t < L; ++t) {
          const uint16_t* vp = d.v_pages + ((d.first_page + (int64_t)b * d.pps + t / P) * d.Hkv + kh) * blk;
          acc += s[t] * bf2f(vp[((int64_t)c * P + t % P) * 8 + i]);
        }
        o[c * 8 + i] = f2bf(acc);
      }
  }
}

#define MGB_AVX512 __attribute__((target("avx512f,avx512bw,avx512vl,avx512dq,avx512bf16")))

// e^x for x <= 0 (softmax arguments): 2^(x log2 e) = 2^n * 2^f, f in [-0.5, 0.5], degree-6 polynomial
// (relative error ~2e-7), scaled with VSCALEFPS (underflows cleanly to 0).
MGB_AVX512 inline __m512 exp512(__m512 x) {
  const __m512 t = _mm512_mul_ps(x, _mm512_set1_ps(1.4426950408889634f));
  const __m512 n = _mm512_roundscale_ps(t, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  const __m512 f = _mm512_sub_ps(t, n);
  __m512 p = _mm512_set1_ps(1.5403530e-4f);
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.3333558e-3f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(9.6181291e-3f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(5.5504109e-2f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(2.4022651e-1f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(6.9314718e-1f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.0f));
  return _mm512_scalef_ps(p, n);
}

// softmax over s[0, L) (s[L, Lp) is padding, zeroed), probabilities rounded to bf16
MGB_AVX512 void softmax_round512(float* s, int L, int Lp, float scale) {
  const __m512 sc = _mm512_set1_ps(scale);
  __m512 m = _mm512_set1_ps(-INFINITY);
  int t = 0;
  for (; t + 16 <= L; t += 16) m = _mm512_max_ps(m, _mm512_mul_ps(_mm512_loadu_ps(s + t), sc));
  float mx = _mm512_reduce_max_ps(m);
  for (; t < L; ++t) mx = std::max(mx, s[t] * scale);
  const __m512 mv = _mm512_set1_ps(mx);
  __m512 sum = _mm512_setzero_ps();
  for (t = 0; t < L; t += 16) {
    const __mmask16 k = L - t >= 16 ? (__mmask16)0xffff : (__mmask16)((1u << (L - t)) - 1);
    const __m512 e = exp512(_mm512_sub_ps(_mm512_mul_ps(_mm512_maskz_loadu_ps(k, s + t), sc), mv));
    const __m512 em = _mm512_maskz_mov_ps(k, e);
    _mm512_mask_storeu_ps(s + t, k, em);
    sum = _mm512_add_ps(sum, em);
  }
  const __m512 inv = _mm512_set1_ps(1.f / _mm512_reduce_add_ps(sum));
  const __m512i rnd = _mm512_set1_epi32(0x7fff), one = _mm512_set1_epi32(1), hi = _mm512_set1_epi32((int)0xffff0000u);
  for (t = 0; t < L; t += 16) {
    const __mmask16 k = L - t >= 16 ? (__mmask16)0xffff : (__mmask16)((1u << (L - t)) - 1);
    const __m512i u = _mm512_castps_si512(_mm512_mul_ps(_mm512_maskz_loadu_ps(k, s + t), inv));
    const __m512i r = _mm512_and_si512(
        _mm512_add_epi32(u, _mm512_add_epi32(rnd, _mm512_and_si512(_mm512_srli_epi32(u, 16), one))), hi);
    _mm512_mask_storeu_ps(s + t, k, _mm512_castsi512_ps(r));  // round to nearest even (finite, >= 0)
  }
  for (t = L; t < Lp; ++t) s[t] = 0.f;
}

MGB_AVX512
void head_avx512(const MgbCpuAttnGqa& d, int b, int kh, std::vector<float>& sc) {
  const int G = d.Hq / d.Hkv, hd = d.hd, P = d.page_tokens, L = d.seq_lens[b], C = hd / 8;
  const int64_t blk = (int64_t)hd * P;
  const int64_t page0 = d.first_page + (int64_t)b * d.pps;
  // q patterns: chunk c of head g repeated for the 4 tokens of one 512-bit K load
  alignas(64) uint16_t qpat[kMaxG][16][32];
  for (int g = 0; g < G; ++g) {
    const uint16_t* q = d.q + ((int64_t)b * d.Hq + kh * G + g) * hd;
    for (int c = 0; c < C; ++c)
      for (int r = 0; r < 4; ++r) memcpy(&qpat[g][c][r * 8], q + c * 8, 16);
  }
  const int Lp = (L + 3) & ~3;
  // ---- scores: 4 tokens x 8 dims per load, VDPBF16PS against the repeated q chunk ----
  for (int t0 = 0; t0 < Lp; t0 += 4) {
    const int p = t0 / P, tt = t0 % P;
    const uint16_t* kp = d.k_pages + (page0 + p) * d.Hkv * blk + (int64_t)kh * blk + (int64_t)tt * 8;
    __m512 acc[kMaxG];
    for (int g = 0; g < G; ++g) acc[g] = _mm512_setzero_ps();
    for (int c = 0; c < C; ++c) {
      const __m512i kv = _mm512_loadu_si512((const void*)(kp + (int64_t)c * P * 8));
      for (int g = 0; g < G; ++g)
        acc[g] = _mm512_dpbf16_ps(acc[g], (__m512bh)kv, (__m512bh)_mm512_load_si512((const void*)qpat[g][c]));
    }
    for (int g = 0; g < G; ++g) {  // lanes 4j..4j+3 hold token t0+j's partial sums
      __m512 v = _mm512_add_ps(acc[g], _mm512_permute_ps(acc[g], 0xB1));
      v = _mm512_add_ps(v, _mm512_permute_ps(v, 0x4E));
      _mm512_mask_storeu_ps(sc.data() + (int64_t)g * Lp + t0 - 0, 0x000f, _mm512_maskz_compress_ps(0x1111, v));
    }
  }
  for (int g = 0; g < G; ++g) softmax_round512(sc.data() + (int64_t)g * Lp, L, Lp, d.scale);
  // ---- PV: blocks of 4 chunks (16 accumulators), two tokens per 512-bit lane set, fp32 FMAs ----
  const __m512i pair_idx = _mm512_set_epi32(1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0);
  for (int c0 = 0; c0 < C; c0 += 4) {
    const int nc = std::min(4, C - c0);
    __m512 acc[kMaxG][4];
    for (int g = 0; g < G; ++g)
      for (int j = 0; j < 4; ++j) acc[g][j] = _mm512_setzero_ps();
    int t = 0;
    for (; t + 1 < L; t += 2) {
      const int p = t / P, tt = t % P;  // t even and P even: t, t+1 share a page
      const uint16_t* vp = d.v_pages + (page0 + p) * d.Hkv * blk + (int64_t)kh * blk + ((int64_t)c0 * P + tt) * 8;
      __m512 pw[kMaxG];
      for (int g = 0; g < G; ++g)
        pw[g] = _mm512_permutexvar_ps(pair_idx, _mm512_castps128_ps512(_mm_castpd_ps(
                                                     _mm_load_sd((const double*)(sc.data() + (int64_t)g * Lp + t)))));
      for (int j = 0; j < nc; ++j) {
        const __m512 v = _mm512_castsi512_ps(_mm512_slli_epi32(
            _mm512_cvtepu16_epi32(_mm256_loadu_si256((const __m256i*)(vp + (int64_t)j * P * 8))), 16));
        for (int g = 0; g < G; ++g) acc[g][j] = _mm512_fmadd_ps(v, pw[g], acc[g][j]);
      }
    }
    for (int g = 0; g < G; ++g)
      for (int j = 0; j < nc; ++j) {
        const int c = c0 + j;
        alignas(64) float o[16];
        _mm512_store_ps(o, acc[g][j]);
        float r[8];
        for (int i = 0; i < 8; ++i) r[i] = o[i] + o[8 + i];
        if (t < L) {  // odd tail
          const int p = t / P, tt = t % P;
          const uint16_t* vp = d.v_pages + (page0 + p) * d.Hkv * blk + (int64_t)kh * blk + ((int64_t)c * P + tt) * 8;
          const float w = sc[(int64_t)g * Lp + t];
          for (int i = 0; i < 8; ++i) r[i] += w * bf2f(vp[i]);
        }
        uint16_t* out = d.out + ((int64_t)b * d.Hq + kh * G + g) * hd + c * 8;
        for (int i = 0; i < 8; ++i) out[i] = f2bf(r[i]);
      }
  }
}

bool have_avx512bf16() {
  static const bool v = !getenv("MGB_CPU_SCALAR") && __builtin_cpu_supports("avx512bf16") && __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512dq") &&
                        __builtin_cpu_supports("avx512vl");
  return v;
}

int run(MgbCpuAttnGqa* d) {
  if (!d || d->B < 1 || d->Hkv < 1 || d->Hq % d->Hkv || d->Hq / d->Hkv > kMaxG || d->hd % 8 || d->hd / 8 > 16 ||
      d->page_tokens % 4 || !d->k_pages || !d->v_pages || !d->q || !d->seq_lens || !d->out) {
    if (d) d->status = -1;
    return -1;
  }
  for (int b = 0; b < d->B; ++b)
    if (d->seq_lens[b] < 1 || d->seq_lens[b] > d->pps * d->page_tokens) {
      d->status = -1;
      return -1;
    }
  const bool fast = have_avx512bf16();
  const int items = d->B * d->Hkv;
  Pool::get().parallel_for(items, [d, fast](int i) {
    thread_local std::vector<float> sc;
    const int b = i / d->Hkv, kh = i % d->Hkv;
    const int Lp = (d->seq_lens[b] + 3) & ~3;
    const size_t need = (size_t)(d->Hq / d->Hkv) * Lp;
    if (sc.size() < need) sc.resize(need);
    if (fast)
      head_avx512(*d, b, kh, sc);
    else
      head_scalar(*d, b, kh, sc);
  });
  d->status = 0;
  return 0;
}

void CUDART_CB host_node(void* p) { run(reinterpret_cast<MgbCpuAttnGqa*>(p)); }

}  // namespace

extern "C" {

// Synchronous CPU attention over the host page store (tests, profiling).
int mgb_cpu_attn_gqa(MgbCpuAttnGqa* desc) { return run(desc); }

// Enqueue the CPU attention as a host node on `stream` (graph-capturable).  `desc` is caller-owned
// and read when the node runs, so it must outlive every replay of a captured graph.
int mgb_cpu_attn_gqa_enqueue(MgbCpuAttnGqa* desc, void* stream) {
  return cudaLaunchHostFunc(reinterpret_cast<cudaStream_t>(stream), host_node, desc) == cudaSuccess ? 0 : -3;
}

// Host threads of the CPU attention pool (default: all hardware threads); returns the pool size.
int mgb_cpu_threads(int n) {
  if (n > 0) Pool::get().resize(n);
  return Pool::get().size();
}

// 1 when the AVX-512 BF16 path is in use on this host.
int mgb_cpu_attn_simd(void) { return have_avx512bf16() ? 1 : 0; }

}  // extern "C"
