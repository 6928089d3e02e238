/*
 * mgb.h — C-ABI of libmgb.so, the B200 (sm_100a) kernels behind the MoE-Gen module-based
 * batching hot path.  Plain pointers + sizes + a cudaStream_t passed as void*; no torch types.
 *
 * The reference (arxiv 2503.09716, /root/reference/pkg) has no operator FFI: its engine-facing
 * interface is the job DAG whose node kinds name the modules the engine launches
 * (pkg/src/moe_planner/offload_dag.py:62-86) and the profiling boundary that names the kernels
 * (pkg/src/moe_planner/hw_profile.py:52-58 ModuleKind).  Each entry point below cites the DAG
 * node / module kind it executes.  Numerics follow HF transformers 5.5.0 (the model definition
 * the paper's engine integrates with).
 *
 * Conventions
 *  - every function returns int: 0 ok, -1 invalid argument, -2 capacity exceeded, -3 CUDA error;
 *  - the caller owns every buffer (device memory unless stated); nothing here allocates HBM;
 *  - all functions are asynchronous on `stream` and reentrant per stream;
 *  - bf16 tensors are row-major, 16-byte aligned rows.
 */
#ifndef MGB_H_
#define MGB_H_

#ifdef __cplusplus
extern "C" {
#endif

/* ---- introspection ---------------------------------------------------------------------- */
int mgb_abi_version(void);
int mgb_num_sms(void);
const char* mgb_last_error(void);
int mgb_kv_page_size(void);                /* tokens per KV page (64) */
int mgb_router_num_blocks(int T);          /* rows of the router block_hist workspace */
int mgb_router_tokens_per_block(void);

/* ---- capacity contract (exec_sim.py:170-175: groups larger than their buffer are split, not
 * overrun; SPEC.md "Invariants": every scheduled row is either processed or reported) ------
 *  - mgb_moe_check_capacity: host pre-flight of a grouped launch whose offsets[E+1] are on the
 *    device: writes per-expert counts to counts_out[E] (host) and returns -2 when the segments need
 *    more than rows_cap rows (the caller re-splits the group by b_e);
 *  - inside a launch (device offsets, graph-replayed steps) the grouped GEMMs and the EP dispatch
 *    check rows_cap on the device, do no out-of-bounds work, and record {-2, rows needed, rows_cap,
 *    site 1 gate/up | 2 down | 3 EP dispatch}; mgb_capacity_status (synchronising) reads it into
 *    out4 (may be NULL), clears it when reset != 0, and returns -2 if an overflow was recorded. */
int mgb_moe_check_capacity(const int* offsets, int E, int rows_cap, int* counts_out, void* stream);
int mgb_capacity_status(int* out4, int reset);

/* ---- ROUTER (offload_dag.py:418-425, ModuleKind.ROUTER hw_profile.py:58) -----------------
 * x[T,d] bf16, w_gate[E,d] bf16 (or logits_in[T,E] fp32 to route given logits).
 * mode 0 Mixtral softmax->topk->renorm; 1 DeepSeek greedy (x scaling); 2 group-limited greedy.
 * Outputs topk_idx[T,k] int32, topk_w[T,k] fp32, counts[E], offsets[E+1]; workspace
 * local_rank[T*k], block_hist[router_num_blocks(T)*E], ticket[1] (zeroed once, self-resetting). */
int mgb_router_topk(const void* x, const void* w_gate, const float* logits_in, int T, int d, int E, int k,
                    int mode, float scaling, int n_group, int topk_group, float* logits_out, int* topk_idx,
                    float* topk_w, int* local_rank, int* block_hist, int* counts, int* offsets, int* ticket,
                    void* stream);

/* ---- fused decode routing front end (route.cu): residual add + RMSNorm (x <- x + delta,
 * h = RMSNorm(x) * ln_w), router logits on the tensor cores, softmax / top-k, counts / offsets and
 * the stable expert-major permutation of h into x_perm -- one launch for ROUTER + the grouping in
 * front of EXPERT_COMPUTE (offload_dag.py:418-463).  chunk_hist: mgb_moe_route_chunks(T) x E ints;
 * sync: 2 ints zeroed once (left reusable).  -1 (and no launch) when T is beyond one co-resident
 * grid (mgb_moe_route_supported); the unfused entry points cover every T.
 * mgb_moe_route_supported: 0 = not covered, 1 = covered, 2 = covered in one pass (one chunk per CTA);
 * h_out may then be NULL (the normalised rows land only in x_perm). */
int mgb_moe_route_chunks(int T);
int mgb_moe_route_stamps(long long* stamps); /* profiling: per-CTA phase globaltimer stamps [G][16], NULL = off */
int mgb_moe_route_supported(int T, int d, int E);
int mgb_moe_route(const void* x, const void* delta, const void* ln_w, float eps, int T, int d, void* x_out,
                  void* h_out, const void* w_router, int E, int k, int mode, float scaling, int n_group,
                  int topk_group, float* logits_out, int* topk_idx, float* topk_w, int* local_rank, int* chunk_hist,
                  int* counts, int* offsets, void* x_perm, int* src_token, int* dst_pos, int* sync, void* stream);

/* ---- token grouping in front of EXPERT_COMPUTE (offload_dag.py:427-463) ------------------
 * Stable expert-major permutation; x_perm[rows_cap,d], src_token[rows_cap], dst_pos[T*k]. */
int mgb_permute(const void* x, const int* topk_idx, const int* local_rank, const int* block_base,
                const int* offsets, int T, int d, int k, int E, void* x_perm, int* src_token, int* dst_pos,
                void* stream);

/* ---- EXPERT_COMPUTE (offload_dag.py:449-463, ModuleKind.EXPERT hw_profile.py:57) ---------
 * tcgen05/TMEM/TMA grouped GEMMs over the expert-major rows; w_gate_up[E,2f,d], w_down[E,d,f]. */
int mgb_moe_gemm_gate_up(const void* w_gate_up, const void* x_perm, const int* offsets, int E, int d, int f,
                         int rows_cap, void* h_out, void* stream);
int mgb_moe_gemm_down(const void* w_down, const void* h, const int* offsets, int E, int d, int f, int rows_cap,
                      void* y_out, void* stream);
/* expert parallelism fused with the data path (peer memory over NVLink, UVA pointers):
 *  - mgb_ep_permute_dispatch: the permutation writes row (t, j) of expert e straight into the owner
 *    rank's receive buffer peer_base[e / E_local] at row disp_row[e] + (position within e's segment);
 *  - mgb_ep_row_ptrs: per receive-buffer row, the home address in the source rank's y_perm
 *    ((local expert, source) segments: start, length, row delta; peer_base = sources' y_perm);
 *  - mgb_moe_gemm_down_ep: the down GEMM whose epilogue stores each row at row_ptr[row] (the combine
 *    send fused into the GEMM). */
int mgb_ep_permute_dispatch(const void* x, const int* topk_idx, const int* local_rank, const int* block_base,
                            const int* offsets, int T, int d, int k, int E, int E_local, const long long* peer_base,
                            const int* disp_row, int recv_rows_cap, int* src_token, int* dst_pos, void* stream);
int mgb_ep_row_ptrs(const int* seg_start, const int* seg_len, const int* seg_delta, int n_seg, int W,
                    const long long* peer_base, int row_bytes, int rows_cap, long long* row_ptr, void* stream);
int mgb_moe_gemm_down_ep(const void* w_down, const void* h, const int* offsets, int E, int d, int f, int rows_cap,
                         const long long* row_ptr, void* stream);
/* The whole expert FFN as ONE persistent tcgen05 CTA-pair launch: gate/up (+ SiLU*up) and down units
 * share one unit list, the down units of expert e waiting on a device counter of e's finished gate/up
 * units (one wave tail, no launch gap).  h_scratch [rows_cap, f]; sync: 257 ints zeroed once (left
 * zero).  Shapes outside the pair tiling (f % 128, d % 256) run the two GEMMs back to back. */
int mgb_moe_ffn(const void* w_gate_up, const void* w_down, const void* x_perm, const int* offsets, int E, int d, int f,
                int rows_cap, void* h_scratch, void* y_out, int* sync, void* stream);
int mgb_grouped_ffn(const void* w_gate_up, const void* w_down, const void* x_perm, const int* offsets, int E, int d,
                    int f, int rows_cap, void* h_scratch, void* y_out, void* stream);

/* ---- combine back to token order (end of the MoE layer, offload_dag.py:465-472) ----------
 * out = residual + bf16(sum_j w*y) (+ shared); optionally norm_out = RMSNorm(out)*norm_w, the
 * next layer's input norm fused in (norm_w/norm_out may be NULL). */
int mgb_unpermute_combine(const void* y_perm, const int* dst_pos, const float* topk_w, const void* shared_out,
                          const void* residual, int T, int d, int k, void* out, const void* norm_w, float eps,
                          void* norm_out, void* stream);

/* ---- ATTN_MECH_GPU (offload_dag.py:393-402, ModuleKind.ATTN_MECH_GPU hw_profile.py:54) ---
 * Paged GQA decode attention; K pages chunk-major, V pages row-major (see attn_gqa.cu). */
int mgb_decode_attn_gqa(const void* q, const void* k_cache, const void* v_cache, const int* block_table,
                        int max_pages, const int* seq_lens, int B, int Hq, int Hkv, int head_dim, float scale,
                        void* out, void* stream);
/* ... with dynamic work-item scheduling: CTAs take (sequence, kv-head) items from a global counter as
 * they stream, so none idles while others finish a static share; sched = 2 ints zeroed once, left
 * zero by every launch (one per stream). */
int mgb_decode_attn_gqa_sched(const void* q, const void* k_cache, const void* v_cache, const int* block_table,
                              int max_pages, const int* seq_lens, int B, int Hq, int Hkv, int head_dim, float scale,
                              void* out, int* sched, void* stream);

/* ... with the step's RoPE + KV append fused in (resident paged KV): qkv [B, (Hq + 2 Hkv) * head_dim]
 * raw projections of the new tokens, positions [B]; rotates q / k (HF rotate_half, cos_t / sin_t
 * [max_pos, head_dim / 2] fp32), writes k / v into each token's page slot and seq_lens[b] =
 * positions[b] + 1, then attends over positions 0..positions[b].  Equals mgb_rope_append_gqa followed
 * by mgb_decode_attn_gqa_sched bit for bit.  Covers PRE_ATTENTION's KV write + ATTN_MECH_GPU
 * (offload_dag.py:359-402).  sched as for mgb_decode_attn_gqa_sched (may be NULL). */
int mgb_decode_attn_gqa_rope(const void* qkv, const int* positions, const float* cos_t, const float* sin_t,
                             void* k_cache, void* v_cache, const int* block_table, int max_pages, int* seq_lens, int B,
                             int Hq, int Hkv, int head_dim, float scale, void* out, int* sched, void* stream);

/* ---- ATTN_MECH_GPU for MLA models (DeepSeek-V2; model_catalog.py:242-295 prices it) -------
 * Absorbed latent attention: q_lat [H,B,R], q_pe [B,H,RP], latent pages of mgb_mla_page_size()
 * tokens and mgb_mla_page_elems(R, RP) bf16 elements, laid out as 64-dim blocks
 * [ceil((R+RP)/64)][page][64] with the 16-byte chunks of each token row 128B-swizzled (chunk c
 * of token t stored at c ^ (t & 7)) -> o_lat [H,B,R].  mgb_mla_append writes the new token's
 * normed latent + RoPE'd k_pe, RoPE's q_pe and re-lays q_nope as [H,B,NOPE]. */
int mgb_mla_page_size(void);
int mgb_mla_page_elems(int R, int RP);
int mgb_decode_attn_mla(const void* q_lat, const void* q_pe, const void* cache, const int* block_table, int max_pages,
                        const int* seq_lens, int B, int H, int R, int RP, float scale, void* o_lat, void* stream);
int mgb_mla_append(const void* q, const void* ckv, const void* norm_w, float eps, int B, int H, int R, int RP, int NOPE,
                   const int* positions, const float* cos_t, const float* sin_t, const int* block_table, int max_pages,
                   void* cache, void* q_nope_out, void* q_pe_out, int* seq_lens, void* stream);
/* prefill (T = n_seq * P prompt tokens, token t = position t % P of sequence seq0 + t / P): latent
 * + k_pe into the pages and into contiguous c_out [T, R] / kpe_out [T, RP]; q_pe rotated in place
 * in q [T, H, NOPE + RP] (for the non-absorbed causal prefill attention) */
int mgb_mla_append_prefill(void* q, const void* ckv, const void* norm_w, float eps, int T, int seq0, int P, int H,
                           int R, int RP, int NOPE, const float* cos_t, const float* sin_t, const int* block_table,
                           int max_pages, void* cache, void* c_out, void* kpe_out, void* stream);

/* ---- prefill attention (the prefill phase's ATTN_MECH_GPU: tokens_per_seq_in_flight = P, no KV
 * copy-in, memory_model.py:53-60, offload_dag.py:359-372) -----------------------------------------
 * Causal attention of n_seq equal-length prompts of P tokens (rows s*P .. s*P+P-1), tcgen05 + TMA
 * (attn_prefill.cu).  q [T, q_cols] head h at column h*q_head_cols; k [T, k_cols] kv head g = h/(Hq/Hkv)
 * at g*k_head_cols (hd_qk - kr_dim dims) + the last kr_dim dims from kr [T, kr_cols] (MLA's shared
 * k_pe; NULL / 0 for GQA); v [T, v_cols] at v_col0 + g*v_head_cols; out [T, out_cols] head h at
 * h*hd_v.  Supported (hd_qk, hd_v): (128, 128), (192, 128), (64, 64) -- mgb_prefill_attn_supported. */
int mgb_prefill_attn_supported(int hd_qk, int hd_v);
int mgb_prefill_attn(const void* q, int q_cols, int q_head_cols, const void* k, int k_cols, int k_head_cols,
                     const void* kr, int kr_cols, int kr_dim, const void* v, int v_cols, int v_head_cols, int v_col0,
                     int n_seq, int P, int Hq, int Hkv, int hd_qk, int hd_v, float scale, void* out, int out_cols,
                     void* stream);

/* ---- KV_COPY_OUT / new-token insert for kv_policy "offload" (offload_dag.py:372-392) --------
 * Copies the token at positions[b] of sequence b from page src_table[b][pos/page_tokens] of src to
 * page dst_table[b][pos/page_tokens] of dst (same in-page slot).  A token's bytes inside a page are
 * n_units runs of unit_bytes, run u at u*unit_stride + slot*unit_bytes (GQA: 16 B / 16*page;
 * MLA: 128 B / 128*page).  src/dst may be mapped pinned host memory (UVA). */
int mgb_kv_token_copy(const void* src, const int* src_table, int src_max_pages, void* dst, const int* dst_table,
                      int dst_max_pages, const int* positions, int B, int page_tokens, long long page_bytes,
                      int unit_bytes, int n_units, long long unit_stride, void* stream);

/* SM-driven byte copy (16 B aligned; either side may be mapped pinned host memory): the CPU share's
 * small per-layer q / length / output transfers, kept off the copy engines the KV slices occupy. */
int mgb_copy_bytes(void* dst, const void* src, long long nbytes, void* stream);

/* ---- ATTN_MECH_CPU (offload_dag.py:328-357; ModuleKind.ATTN_MECH_CPU hw_profile.py:55) -----
 * GQA decode attention on the host cores over the host KV page store (GPU page layout), for the
 * plan's CPU share of sequences (omega > 0).  AVX-512 BF16 when the host has it, scalar otherwise.
 * mgb_cpu_attn_gqa runs synchronously; mgb_cpu_attn_gqa_enqueue adds it to `stream` as a host node
 * (cudaLaunchHostFunc; CUDA-graph capturable) and reads `desc` when the node runs. */
typedef struct MgbCpuAttnGqa {
  const unsigned short* k_pages; /* host page store of the layer, K (bf16 bits) */
  const unsigned short* v_pages; /* V */
  const unsigned short* q;       /* [B, Hq, hd] bf16, RoPE applied (pinned host) */
  const int* seq_lens;           /* [B] keys per sequence (pinned host) */
  unsigned short* out;           /* [B, Hq * hd] bf16 (pinned host) */
  long long first_page;          /* sequence b owns pages first_page + b * pps ... */
  int pps, B, Hq, Hkv, hd, page_tokens;
  float scale;
  int status;                    /* written by the host node: 0 ok, -1 invalid */
} MgbCpuAttnGqa;
int mgb_cpu_attn_gqa(MgbCpuAttnGqa* desc);
int mgb_cpu_attn_gqa_enqueue(MgbCpuAttnGqa* desc, void* stream);
int mgb_cpu_threads(int n);        /* resize the host thread pool (n > 0); returns its size */
int mgb_cpu_attn_simd(void);       /* 1 if the AVX-512 BF16 path is active */

/* ---- PRE_ATTENTION / POST_ATTENTION helpers (offload_dag.py:359-416) --------------------- */
int mgb_add_rmsnorm(const void* x, const void* delta, const void* weight, float eps, int T, int d, void* x_out,
                    void* y, void* stream);
int mgb_rope_append_gqa(const void* qkv, int T, int seq0, const int* positions, const float* cos_t,
                        const float* sin_t, int Hq, int Hkv, int head_dim, const int* block_table, int max_pages,
                        void* k_cache, void* v_cache, void* q_out, int* seq_lens, void* stream);
/* prefill (T = n_seq * P prompt tokens, token t = position t % P of sequence seq0 + t / P): RoPE'd q
 * to q_out, K/V into the pages and into contiguous k_out / v_out [T, Hkv, hd] for the causal attention */
int mgb_rope_append_gqa_prefill(const void* qkv, int T, int seq0, int P, const float* cos_t, const float* sin_t,
                                int Hq, int Hkv, int head_dim, const int* block_table, int max_pages, void* k_cache,
                                void* v_cache, void* q_out, void* k_out, void* v_out, void* stream);
int mgb_embed(const int* ids, const void* table, int T, int d, void* out, void* stream);
/* h[T,F] = bf16(bf16(silu(g)) * u) for gate_up[T, 2F] = [g | u] (dense/shared-expert MLP epilogue) */
int mgb_silu_mul(const void* gate_up, int T, int F, void* h, void* stream);
int mgb_argmax(const void* logits, int T, int V, int* out, void* stream);
int mgb_decode_advance(const int* next, int B, long long* out_tokens, int ld, int* step, int* positions,
                       void* stream);

/* ---- synthetic random-init weights (counter-based, mirrored by oracle/rng.py) ------------ */
int mgb_fill_uniform_bf16(void* out, long long n, unsigned long long seed, unsigned long long tensor_id, float std,
                          float constant, int mode, void* stream);
/* elements [first, first + n) of the same stream (a rank's expert shard, generated in place) */
int mgb_fill_uniform_bf16_range(void* out, long long n, long long first, unsigned long long seed,
                                unsigned long long tensor_id, float std, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MGB_H_ */
