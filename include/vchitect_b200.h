/*
 * vchitect_b200.h -- C ABI of the B200-native parallel MM-DiT block forward.
 *
 * Drop-in boundary for the hot path of arXiv 2501.08453 (Vchitect-2.0) as
 * implemented by the reference CPU simulator `spsim`. Every entry point below
 * names the reference function it replaces (paths relative to
 * /root/reference/pkg/src/spsim/). The reference is a Python/numpy API with
 * no FFI; the binding a maintainer would add on the reference side (ctypes)
 * is shown in INTEGRATION.md.
 *
 * Conventions
 *   - Plain pointers and sizes only. "dev" pointers are CUDA device memory,
 *     "host" pointers are host memory (pinned for async copies).
 *   - Every call is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*), never synchronises the device, never allocates device memory:
 *     callers own the weight and workspace buffers (sizes from *_bytes()).
 *   - Return VC_OK (0) or a negative code; vc_last_error() gives a message
 *     (thread-local). Shape / divisibility violations return VC_EINVAL with
 *     the reference's ValueError wording.
 *   - Thread-safe across distinct streams and buffers.
 *   - Weight layout in (`raw`) is the reference's BranchParams layout:
 *     per branch gamma[D], beta[D], wq, wk, wv, wo each [D_in][D_out]
 *     row-major (applied as x @ W, model.py:157-184); a block is the three
 *     branches in order spatial, temporal, fullseq (model.py:193-205).
 */
#ifndef VCHITECT_B200_H
#define VCHITECT_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define VC_API __attribute__((visibility("default")))
#else
#define VC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define VC_OK 0
#define VC_EINVAL (-22)
#define VC_ECUDA (-1000)
#define VC_ENOTSUP (-95)

/* arithmetic of the path: fp32 (SIMT FFMA, the 1e-4 parity path) or bf16
 * operands with fp32 accumulation on tcgen05 tensor cores. */
#define VC_DTYPE_F32 0
#define VC_DTYPE_BF16 1

typedef struct vc_block_shape {
  int32_t frames;     /* F  */
  int32_t visual_len; /* Lv visual tokens per frame */
  int32_t text_len;   /* Lt prompt tokens (anchored to every frame) */
  int32_t dim;        /* D  */
  int32_t heads;      /* H, D % H == 0 */
  int32_t dtype;      /* VC_DTYPE_* */
} vc_block_shape;

/* Library build/version string, e.g. "vchitect_b200 sm_100a ...". */
VC_API const char* vc_version(void);

/* Message of the last failing call on this thread. */
VC_API const char* vc_last_error(void);

/* Validate a shape (model.py:263-271 preconditions; numerics.py:93-99). */
VC_API int vc_block_shape_check(const vc_block_shape* shape);

/* Element count of one block's raw fp32 weights: 3 * (2*D + 4*D*D). */
VC_API size_t vc_block_raw_weight_floats(const vc_block_shape* shape);

/* Bytes of one block's packed device weights (gamma folded into W,
 * beta@W bias, Q/K/V of the three branches concatenated, O weights stacked). */
VC_API size_t vc_block_packed_weight_bytes(const vc_block_shape* shape);

/* Bytes of device workspace vc_block_forward needs. */
VC_API size_t vc_block_workspace_bytes(const vc_block_shape* shape);

/* Pack raw fp32 device weights (reference layout, see above) into the
 * device layout the kernels consume. Replaces nothing in the reference
 * (weights are used as-is there); it is the one-time load step. */
VC_API int vc_pack_block_weights(const vc_block_shape* shape, const float* raw_dev,
                          void* packed_dev, void* stream);

/* Block forward.  Replaces parallel_block_forward (model.py:263-271) and,
 * with add_residual=1, one iteration of ToyDenoiser.head_states'
 * `x = x + block(x)` (model.py:323-324).
 *   visual_dev [F][Lv][D] fp32, prompt_dev [Lt][D] fp32 (= text[0]; the
 *   reference anchors every frame's text slots to it, model.py:257),
 *   out_dev [F][Lv][D] fp32 (may alias visual_dev when add_residual=1). */
VC_API int vc_block_forward(const vc_block_shape* shape, const void* packed_dev,
                     const float* visual_dev, const float* prompt_dev,
                     float* out_dev, int add_residual, void* workspace_dev,
                     size_t workspace_bytes, void* stream);

/* Same as vc_block_forward with HOST buffers: copies visual/prompt in,
 * runs, copies out back, all on `stream` (the call does not synchronise;
 * the caller syncs before reading out_host). Staging buffers for the
 * device-side copies are carved from the workspace; size with
 * vc_block_host_workspace_bytes(). */
VC_API size_t vc_block_host_workspace_bytes(const vc_block_shape* shape);
VC_API int vc_block_forward_host(const vc_block_shape* shape, const void* packed_dev,
                          const float* visual_host, const float* prompt_host,
                          float* out_host, void* workspace_dev,
                          size_t workspace_bytes, void* stream);

/* Streamed host path: n block forwards of HOST batches visual_host[i]
 * ([F][Lv][D] fp32, pinned) sharing one prompt, results to out_host[i].
 * Double-buffered: the H2D of batch i+1 and the D2H of batch i-1 run on
 * h2d_stream / d2h_stream while batch i computes on compute_stream, so a
 * serving loop runs at max(compute, PCIe in, PCIe out) per batch. Work
 * queued on compute_stream completes after the last copy out. */
VC_API size_t vc_block_stream_workspace_bytes(const vc_block_shape* shape);
VC_API int vc_block_forward_host_batched(const vc_block_shape* shape,
                                         const void* packed_dev, int32_t n,
                                         const float* const* visual_host,
                                         const float* prompt_host,
                                         float* const* out_host,
                                         void* workspace_dev,
                                         size_t workspace_bytes,
                                         void* compute_stream, void* h2d_stream,
                                         void* d2h_stream);

/* Multi-head attention, numerics.py:87-107: q [sq][D], k/v [sk][D] fp32
 * device, heads contiguous column slices, scale 1/sqrt(D/heads), non-causal.
 * fp32 SIMT path (parity 1e-4 class). */
VC_API int vc_attention_f32(const float* q_dev, const float* k_dev, const float* v_dev,
                     float* out_dev, int32_t sq, int32_t sk, int32_t dim,
                     int32_t heads, void* stream);

/* The same attention on tcgen05 tensor cores (bf16 operands, fp32
 * accumulation; the kernels the block forward runs), plus the deduplicated-
 * text form of the full-sequence branch: the first n_weighted keys carry a
 * multiplicity key_weight (logit + log key_weight), e.g. the F identical
 * anchored prompt copies (model.py:257) as one key each with weight F.
 * Head dims up to 128 (padded to 64 / 80 / 128). Device workspace of
 * vc_attention_bf16_workspace_bytes() bytes. bf16 parity class (2e-2). */
VC_API size_t vc_attention_bf16_workspace_bytes(int32_t sq, int32_t sk, int32_t dim,
                                                int32_t heads);
VC_API int vc_attention_bf16(const float* q_dev, const float* k_dev, const float* v_dev,
                             float* out_dev, int32_t sq, int32_t sk, int32_t dim,
                             int32_t heads, int32_t n_weighted, float key_weight,
                             void* workspace_dev, size_t workspace_bytes, void* stream);

/* LayerNorm without affine, model.py:89-92 (biased var, eps 1e-5):
 * rows x [rows][D] fp32 -> out fp32. */
VC_API int vc_layer_norm_f32(const float* x_dev, float* out_dev, int64_t rows,
                      int32_t dim, void* stream);

/* ToyDenoiser.embed_frame for all frames, model.py:303-314 + patchify
 * model.py:53-64: latents [F][h][w][c] fp32, w_in [p*p*c][D] fp32 ->
 * x [F][Lv][D] fp32 (+ sinusoid of global token index (first_frame+f)*Lv+i
 * and of t). */
VC_API int vc_embed_frames(const float* latents_dev, const float* w_in_dev,
                    float* x_dev, int32_t frames, int32_t first_frame,
                    int32_t h, int32_t w, int32_t c, int32_t patch,
                    int32_t dim, double t, void* stream);

/* toy_vae_encode (model.py:381-403) of F frames [F][H][W][3] fp32 ->
 * latents [F][ceil(H/d)][ceil(W/d)][channels] fp32 (zero-padded d x d block
 * average, fixed cosine channel mix), optionally with q_sample
 * (diffusion.py:77-84) fused: latents = sqrt_alpha_bar * encode +
 * sqrt_one_minus_alpha_bar * noise (noise [F][gh][gw][channels]; NULL for the
 * plain encode: pass 1, 0). channels <= 16. */
VC_API int vc_vae_encode_frames(const float* pixels_dev, const float* noise_dev, float* latents_dev, int32_t F,
                                int32_t H, int32_t W, int32_t downsample, int32_t channels, double sqrt_alpha_bar,
                                double sqrt_one_minus_alpha_bar, void* stream);

/* Row subset of vc_embed_frames: tokens [tok0, tok0+ntok) of every frame ->
 * x [F][ntok][D]. A sequence-parallel rank embeds its own rows directly
 * (the embedding is position-wise), replacing the reference's frame-wise
 * embed + all-to-all reshard (executor.py:535-559) with no communication. */
VC_API int vc_embed_frames_rows(const float* latents_dev, const float* w_in_dev,
                                float* x_dev, int32_t frames, int32_t first_frame,
                                int32_t tok0, int32_t ntok, int32_t h, int32_t w,
                                int32_t c, int32_t patch, int32_t dim, double t,
                                void* stream);

/* ToyDenoiser.forward's output projection + unpatchify crop,
 * model.py:331-333 + model.py:67-76: x [F][Lv][D], w_out [D][p*p*c] ->
 * eps [F][h][w][c] fp32. */
VC_API int vc_unembed_frames(const float* x_dev, const float* w_out_dev,
                      float* eps_dev, int32_t frames, int32_t h, int32_t w,
                      int32_t c, int32_t patch, int32_t dim, void* stream);

/* One denoise step, output side: the unembed of vc_unembed_frames with the
 * DDPM ancestral step reverse_step (diffusion.py:95-116) fused into its
 * epilogue: x_prev = (x_t - coef_eps * eps) * inv_sqrt_alpha
 * (+ sqrt_beta * noise when noise != NULL), coef_eps = beta_t /
 * sqrt(1 - alpha_bar_t), inv_sqrt_alpha = 1 / sqrt(alpha_t) (host fp64 from
 * the schedule). eps may be NULL (not stored). All [F][h][w][c] fp32. */
VC_API int vc_unembed_reverse_step(const float* x_dev, const float* w_out_dev,
                                   const float* x_t_dev, const float* noise_dev,
                                   float* eps_dev, float* x_prev_dev,
                                   int32_t frames, int32_t h, int32_t w, int32_t c,
                                   int32_t patch, int32_t dim, double coef_eps,
                                   double inv_sqrt_alpha, double sqrt_beta,
                                   void* stream);

/* The tcgen05 GEMM on its own: out[m][n] = sum_k A[m][k] B[n][k]
 * (+ bias[n]) (+ resid[m][n]), A/B bf16 K-major (row pitch lda/ldb elements,
 * 16-byte aligned), fp32 accumulation and output. The projection GEMMs of the
 * block (model.py:184, :190) run through this kernel with fused epilogues. */
VC_API int vc_gemm_bf16(const void* a_dev, int64_t lda, const void* b_dev,
                        int64_t ldb, const float* bias_dev,
                        const float* resid_dev, float* out_dev, int64_t ldo,
                        int64_t M, int32_t N, int32_t K, void* stream);

/* Temporal-branch kernel choice for the bf16 block (test / profiling aid):
 * 0 the measured rule (default: the tcgen05 + TMA kernel on 64..128-frame,
 * dh >= 128 sequences, the mma.sync kernel elsewhere), 1 mma.sync, 2 the
 * tcgen05 + TMA kernel wherever it applies (F <= 176, dh <= 128).
 * Process-wide; not thread-safe against concurrent forwards. */
VC_API int vc_set_temporal_impl(int32_t impl);

/* ---- Sequence parallelism (the paper's hybrid-parallel scheme) ----------
 * Spatial shard axis, head-parallel (Ulysses) attention, separate text
 * placement: executor.py:561-626 (run_sp_iteration stage 3) with the two
 * all-to-alls of _branch_head_parallel (executor.py:332-413). Rank r holds
 * visual rows [vb[r], vb[r+1]) of every frame, vb = contiguous_bounds(Lv, P)
 * (executor.py:187-191), and the whole prompt. The host runs
 *   stage1 -> all_to_all(send1 -> recv1) -> stage2 -> all_to_all(send2 ->
 *   recv2) -> stage3
 * with per-peer counts from vc_sp_exchange_elems (bf16 elements). bf16 only.
 * All four buffers are BRANCH-MAJOR: the first half holds the spatial
 * branch for every peer, the second half the full-sequence branch, each half
 * split by peer with half the per-peer count. So the exchange can run per
 * branch and overlap compute: stage1 -> a2a#1(spatial), a2a#1(full seq) ->
 * wait spatial -> stage2_branch(0) -> a2a#2(spatial) -> wait full seq ->
 * stage2_branch(1) -> a2a#2(full seq) -> wait -> stage3. */
typedef struct vc_sp_plan {
  vc_block_shape shape; /* global block shape (dtype must be VC_DTYPE_BF16) */
  int32_t nranks;       /* P: sp_size */
  int32_t rank;
} vc_sp_plan;

/* executor.py:517-529 validity: P <= Lv, H % P == 0 (P > 1). */
VC_API int vc_sp_check(const vc_sp_plan* plan);
/* vbounds[0..P] = contiguous_bounds(Lv, P) (executor.py:187-191). */
VC_API int vc_sp_bounds(const vc_sp_plan* plan, int32_t* vbounds);
VC_API size_t vc_sp_workspace_bytes(const vc_sp_plan* plan);
/* Frame-wise -> spatial reshard (alltoall_reshard, executor.py:252-287,
 * spatial axis): rank d holds the embedded frames f = d, d+P, ... (the
 * round-robin deal, executor.py:194-196) as [n_d][Lv][D] fp32; pack writes
 * the send buffer (peer r gets rows [vb[r], vb[r+1]) of each), all_to_all,
 * unpack writes the resident [F][vc_rank][D]. which 0: send elements to
 * peer, 1: receive elements from peer (fp32). Resident equal to
 * allgather_then_shard (executor.py:290-308) exactly. */
VC_API int64_t vc_sp_reshard_elems(const vc_sp_plan* plan, int32_t which, int32_t peer);
VC_API int vc_sp_reshard_pack(const vc_sp_plan* plan, const float* local_frames, float* send, void* stream);
VC_API int vc_sp_reshard_unpack(const vc_sp_plan* plan, const float* recv, float* resident, void* stream);

/* The row maps the exchanges use (exact-equality tests against the
 * reference's stable argsort, executor.py:349-370, :606-617). which 0: for
 * the rows of every rank concatenated in rank order (each rank's local rows
 * frame-major), the visual token f*Lv + l the a2a #1 unpack assembles them
 * as (F*Lv entries); which 1: for each visual token, the index of the row it
 * is returned to by a2a #2 in that same concatenation. Host only. */
VC_API int vc_sp_row_map(const vc_sp_plan* plan, int32_t which, int64_t* out);
/* which: 0 send1 to peer, 1 recv1 from peer, 2 send2 to peer, 3 recv2 from
 * peer (bf16 elements as laid out: head dim padded to DP, dh-66 outputs in
 * DP-wide head slots; 0 for peer == rank: the own block never enters the
 * buffers, stage 1 / 2 write it straight where stage 2 / 3 read it); 4..7
 * the reference's payload (executor.py:344-347, :395-412): no padding, own
 * block included. -1 on error. */
VC_API int64_t vc_sp_exchange_elems(const vc_sp_plan* plan, int32_t which,
                                    int32_t peer);
/* x_local [F][vc_r][D] fp32, prompt [Lt][D] fp32 -> send1 (bf16). */
VC_API int vc_sp_stage1(const vc_sp_plan* plan, const void* packed_dev,
                        const float* x_local_dev, const float* prompt_dev,
                        void* send1_dev, void* workspace_dev,
                        size_t workspace_bytes, void* stream);
/* vc_sp_stage1 in two parts, so the host can start a2a #1 after the QKV GEMM
 * and run the rank-local temporal branch under it: part 0 = LN + QKV GEMM
 * (fills send1), 1 = temporal branch, 2 = both (= vc_sp_stage1). */
VC_API int vc_sp_stage1_part(const vc_sp_plan* plan, const void* packed_dev, const float* x_local,
                             const float* prompt, void* send1, int32_t part, void* workspace,
                             size_t workspace_bytes, void* stream);
/* One branch of stage 2 (0 spatial, 1 full sequence): that branch's half of
 * recv1 -> head-group attention -> that branch's half of send2. */
VC_API int vc_sp_stage2_branch(const vc_sp_plan* plan, const void* packed_dev,
                               const void* recv1_dev, void* send2_dev, int32_t branch,
                               void* workspace_dev, size_t workspace_bytes,
                               void* stream);
/* recv1 -> head-group attention -> send2 (bf16); both branches. */
VC_API int vc_sp_stage2(const vc_sp_plan* plan, const void* packed_dev,
                        const void* recv1_dev, void* send2_dev,
                        void* workspace_dev, size_t workspace_bytes,
                        void* stream);
/* recv2 -> O projection (+ x_local if add_residual) -> out_local fp32. */
VC_API int vc_sp_stage3(const vc_sp_plan* plan, const void* packed_dev,
                        const void* recv2_dev, const float* x_local_dev,
                        float* out_local_dev, int add_residual,
                        void* workspace_dev, size_t workspace_bytes,
                        void* stream);

/* ---- Gather-mode sequence parallelism -----------------------------------
 * _branch_gather (executor.py:416-459), the plan.attention != "head_parallel"
 * branch of _run_branch (:462-466): every rank all-gathers the spatial and
 * full-sequence K,V of ALL heads and attends for its own rows, so P need not
 * divide H (e.g. 4 heads on 8 ranks). Same shard map as above. The host runs
 *   vc_spg_stage1 (writes this rank's slot of the gather buffer)
 *   -> all_gather (vc_spg_slot_elems bf16 per rank, slot r at r*slot_elems)
 *   -> vc_spg_stage2
 * Exchange per rank: (P-1)/P of 4*Nv*D-ish bf16 (K,V of two branches), about
 * 4x the head-parallel volume — head-parallel stays the default when H % P == 0. */
/* validity: P <= Lv (executor.py:521-524), 1..16 ranks. */
VC_API int vc_spg_check(const vc_sp_plan* plan);
VC_API size_t vc_spg_workspace_bytes(const vc_sp_plan* plan);
/* bf16 elements of one rank's slot (identical for every rank); -1 on error. */
VC_API int64_t vc_spg_slot_elems(const vc_sp_plan* plan);
/* x_local [F][vc_r][D] fp32, prompt [Lt][D] fp32 -> this rank's K,V slot
 * (gather + rank * slot_elems); the local Q, the temporal branch and the
 * text K,V of all heads (from the local prompt copy) stay in the workspace. */
VC_API int vc_spg_stage1(const vc_sp_plan* plan, const void* packed_dev,
                         const float* x_local_dev, const float* prompt_dev,
                         void* gather_dev, void* workspace_dev,
                         size_t workspace_bytes, void* stream);
/* gathered K,V of all ranks -> attention of the local rows (all heads) ->
 * O projection (+ x_local if add_residual) -> out_local fp32. */
VC_API int vc_spg_stage2(const vc_sp_plan* plan, const void* packed_dev,
                         const void* gather_dev, const float* x_local_dev,
                         float* out_local_dev, int add_residual,
                         void* workspace_dev, size_t workspace_bytes,
                         void* stream);

/* Stage profiler (bench accounting, not used on the timed path): when
 * enabled, vc_block_forward records a CUDA event after each of its kernels,
 * synchronises at the end of the call and accumulates per-stage device time
 * by stage name ("ln", "qkv_gemm", "attn_spatial", ...). */
VC_API int vc_profile_enable(int on);
VC_API void vc_profile_reset(void);
/* Fills up to max_stages entries; names is a '\n'-joined list written into
 * names_buf. Returns the number of stages. */
VC_API int vc_profile_read(double* ms_total, int32_t* calls, int32_t max_stages,
                           char* names_buf, size_t names_len);

/* Number of kernel launches vc_block_forward issues for `shape` (the
 * bench's gpu_launches accounting). */
VC_API int vc_block_forward_launches(const vc_block_shape* shape);

/* ---- north-star extensions (no reference counterpart; PARITY UNPINNED) ----
 * BASELINE.json's north_star names pieces of the Vchitect-2.0 block that the
 * reference spsim block (model.py:263-271) lacks (SURVEY.md §8 "a-ext"):
 * AdaLN timestep modulation, QK-RMSNorm + 3D RoPE fused into the Q/K
 * projection epilogue, the gated residual and the gated GELU FFN.  Their
 * semantics are defined by oracle/vchitect_ext_oracle.py:
 *   mod = silu(sinusoidal_embedding(t, D)) @ w_ada + b_ada   -> 6 x [D]
 *   h = x + gate_msa * block'(LN(x) * (1 + scale_msa) + shift_msa)
 *   y = h + gate_mlp * (gelu_tanh(n2 @ w1 + b1) @ w2 + b2),
 *       n2 = LN(h) * (1 + scale_mlp) + shift_mlp
 * where block' is the reference block with RMSNorm + RoPE on the spatial and
 * full-sequence Q/K heads.  bf16 only; the reference-semantics entry points
 * above are unchanged by any of this. */
typedef struct vc_ext_shape {
  vc_block_shape block;   /* dtype must be VC_DTYPE_BF16, head dim even */
  int32_t grid_h, grid_w; /* patch grid, grid_h * grid_w == visual_len (RoPE rows / columns) */
  int32_t ffn_dim;        /* FFN hidden width (mlp_ratio * D), multiple of 8 */
} vc_ext_shape;

/* Raw fp32 extension weights, concatenated: w_ada [D][6D], b_ada [6D],
 * q_norm [2][dh], k_norm [2][dh] (rows: spatial, full sequence),
 * w1 [D][ffn], b1 [ffn], w2 [ffn][D], b2 [D] (x @ W layout). */
VC_API size_t vc_ext_raw_weight_floats(const vc_ext_shape* shape);
VC_API size_t vc_ext_packed_weight_bytes(const vc_ext_shape* shape);
VC_API int vc_pack_ext_weights(const vc_ext_shape* shape, const float* raw_dev, void* packed_dev,
                               void* stream);
VC_API size_t vc_ext_workspace_bytes(const vc_ext_shape* shape);
/* y = extended block(visual, prompt, timestep); block_packed_dev from
 * vc_pack_block_weights (bf16), out_dev must not alias visual_dev. */
VC_API int vc_ext_block_forward(const vc_ext_shape* shape, const void* block_packed_dev,
                                const void* ext_packed_dev, const float* visual_dev,
                                const float* prompt_dev, double timestep, float* out_dev,
                                void* workspace_dev, size_t workspace_bytes, void* stream);
VC_API int vc_ext_block_launches(const vc_ext_shape* shape);

#ifdef __cplusplus
}
#endif

#endif /* VCHITECT_B200_H */
