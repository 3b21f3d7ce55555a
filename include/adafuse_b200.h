/*
 * adafuse_b200.h -- C ABI of the B200-native AdaFuse hot path.
 *
 * The reference (`lorafuse`, pure Python/numpy) has no FFI of its own;
 * the boundary it exposes is its Python call surface.  Each entry point below names the
 * reference function it replaces (paths relative to /root/reference/pkg/src/lorafuse/).
 * The Python host (`paper_2603_11873_b200`) binds these with ctypes; INTEGRATION.md shows
 * the stub a maintainer of the reference would add.
 *
 * Conventions
 *   - plain pointers and sizes only; every device buffer is OWNED BY THE CALLER
 *     (the library owns only the table objects it creates and their TMA maps);
 *   - every call returns an int status (AF_OK == 0); no exceptions, no aborts; the
 *     message of the last failure on this thread is af_last_error();
 *   - validation happens BEFORE any data is touched (linalg.py:323-325, routing.py:57-62);
 *   - all work is enqueued on the caller's `stream` (a cudaStream_t passed as void*);
 *     no call synchronises unless it says so;
 *   - matrices are row-major; `ld` is the row pitch in ELEMENTS.
 */
#ifndef ADAFUSE_B200_H
#define ADAFUSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AF_ABI_VERSION 3

/* ---- status codes: one per reference exception class (errors.py:8-33) ---- */
#define AF_OK 0
#define AF_EVALUE 1      /* ValueError      bad sign / k / enum                       */
#define AF_EDIM 2        /* DimensionError  shapes disagree, empty table               */
#define AF_EPRECISION 3  /* PrecisionError  unsupported / mixed dtype tags             */
#define AF_EALIAS 4      /* AliasingError   two segments share / overlap one target    */
#define AF_EINPUT 5      /* InputError      token outside the vocabulary               */
#define AF_ESTATE 6      /* StateError      missing state (no pristine copy, ...)      */
#define AF_EINDEX 7      /* IndexError      expert id outside the bank                 */
#define AF_ECUDA 8       /* a CUDA runtime/driver call failed (message has the code)   */

/* ---- element types ---- */
#define AF_BF16 0
#define AF_F32 1

/* ---- fused-switch options ---- */
#define AF_SWITCH_INPLACE 0       /* W <- W + dNew - dOld   (model.py:350-357)            */
#define AF_SWITCH_FROM_PRISTINE 1 /* W <- W0 + dNew         (refresh, model.py:308-312, fused with the merge) */

#define AF_COMPUTE_AUTO 0  /* library picks FMA or MMA from the effective rank          */
#define AF_COMPUTE_EXACT 1 /* reference order: per rank (mul, round)(add, round); bit-exact vs linalg.py:338-343 in f32 */
#define AF_COMPUTE_FMA 2   /* f32 FMA on CUDA cores, repeated experts collapsed         */
#define AF_COMPUTE_MMA 3   /* B.(g*A) on the tensor pipe: g*A kept f32-accurate as a bf16 hi+lo pair, f32 accumulate */

#define AF_MAX_K 8 /* experts per decision (top-k <= 8) */

/* GEMV epilogues */
#define AF_EPI_NONE 0
#define AF_EPI_GELU_RESIDUAL 1 /* out = res + 0.5*y*(1+erf(y/sqrt2))   (model.py:298,305) */
#define AF_EPI_RESIDUAL 2      /* out = res + y                                          */

/* routing.py:37-46 `GateDecision`, device/host POD form.  ids ordered by descending
 * logit, ties by ascending index; weights > 0, sum to 1 (f32). */
typedef struct af_decision {
    int32_t k;
    int32_t ids[AF_MAX_K];
    float weights[AF_MAX_K];
    int32_t reserved[15]; /* pads the record to 128 bytes */
} af_decision;

/* linalg.py:183-217 `Segment`, as addresses.  One adapted matrix and the factors that
 * can update it.  Two uses:
 *   bank form        (adapters.py:71-109 `ExpertBank`): down = [N][rank][d_in],
 *                    up = [N][d_out][rank]; the per-token (expert, weight) list selects blocks;
 *   materialised form (adapters.py:117-162 `ConcatAdapter`): n_experts = 1,
 *                    down = s x d_in, up = d_out x s, rank = s. */
typedef struct af_segment_desc {
    void* target;         /* d_out x d_in, mutated in place (linalg.py:336-343)          */
    const void* pristine; /* optional untouched copy (model.py:153), same shape/pitch    */
    const void* down;     /* LoraExpert.down blocks (adapters.py:53)                      */
    const void* up;       /* LoraExpert.up blocks   (adapters.py:54)                      */
    int32_t d_out;
    int32_t d_in;
    int32_t rank;         /* rows of one down block; 0 is legal (no-op, linalg.py:190)    */
    int32_t n_experts;
    int64_t ld_target;    /* elements                                                    */
    int64_t ld_down;      /* row pitch of a down block (elements)                        */
    int64_t ld_up;        /* row pitch of an up block (elements)                         */
    int64_t down_expert_stride; /* elements between consecutive experts' down blocks      */
    int64_t up_expert_stride;   /* elements between consecutive experts' up blocks        */
} af_segment_desc;

typedef struct af_table af_table; /* linalg.py:207-231 `SegmentTable`, device resident */

/* ---- library ---- */
int af_abi_version(void);
const char* af_last_error(void);
/* Fills what the caller asks for (any pointer may be NULL). */
int af_device_info(int* sm_count, int* cc_major, int* cc_minor, int64_t* l2_bytes);
/* Number of kernel launches issued by this library since load (bench `gpu_launches`). */
int64_t af_launch_count(void);
/* Name (template arguments included) of the switch kernel the calling thread's last af_fused_switch /
 * af_merge / af_unmerge / af_sgmm / af_switch_gemv[_chain] call launched -- what a benchmark reports. */
const char* af_last_switch_kernel(void);
/* Programmatic dependent launch of the decode GEMV / attention chain (default on; the
 * environment variable AF_PDL=0 turns it off at load).  With it, a GEMV prefetches its first
 * weight tiles while the previous kernel of the stream is still draining. */
int af_set_pdl(int32_t enable);
/* Streaming strategy of af_gemv_fused: 0 = through registers (LDG.128), 1..4 = through a
 * shared-memory ring filled by 1-D bulk copies (copy size / producer threads: 2 KB x1, 2 KB x2,
 * 4 KB x1, 4 KB x2); full_sm != 0 lets the ring take the whole SM instead of half of it.
 * Results are identical up to f32 summation order.  Env: AF_GEMV, AF_GEMV_FULL_SM. */
int af_set_gemv_variant(int32_t variant, int32_t full_sm);
/* Tensor path of the fused switch (+ GEMV) on eligible tables (one rank in {8, 16, 32, 64} everywhere,
 * every matrix at least 128 x 128 with rows a multiple of 8; launches of up to 256 stacked ranks):
 * 1 = tcgen05.mma with the accumulators in tensor memory (csrc/af_switch_umma.cuh; default),
 * 0 = mma.sync kernels (what every other table and launch uses).
 * Both are within 1 bf16 ulp of the f32 merge; they round differently in the last bit, so do not mix
 * them inside one comparison.  Env: AF_UMMA=0 turns the tcgen05 path off at load;
 * AF_UMMA_MAX_RANKS / AF_UMMA_MAX_RANKS_CHAIN move the limits (A/B runs). */
int af_set_umma(int32_t enable);
/* bf16 pieces the tcgen05 kernels split a gated DOWN row (g * a, an f32 value) into before the tensor cores
 * multiply it with UP: 2 (default; g*a reproduced to 2^-17 relative, as the mma.sync kernels do) or 3 (g*a exact --
 * 24 bits in three 8-bit pieces -- so the merge differs from the reference's f32 `B @ (g*A)` of linalg.py:150-168
 * only by the order of the f32 sums: 8x fewer last-bit differences against the oracle at Llama-2-7B, for 0.4 % of the
 * step at full clocks and 1.5 % on a power-capped board -- 50 % more tensor work).  Three pieces apply to launches of
 * at most 32 stacked ranks (rank 8, top-2: BASELINE configs[0..1] and [3]); larger launches always use two (the slab
 * would cost a ring stage).  The two settings round differently in the last bit: do not mix them inside one
 * comparison.  AF_EVALUE for anything but 2 or 3.  Env: AF_UMMA_PIECES. */
int af_set_umma_pieces(int32_t pieces);

/* ---- segment table: built once at model load -------------------------------------
 * Replaces: linalg.py:207-231 `SegmentTable` + `.validate()` (shape, precision and
 * distinct-target checks) and the per-token Segment construction of adapters.py:252-257.
 * Builds the device-side descriptor table (segments + work units) and one TMA tensor
 * map per segment.  Errors: AF_EDIM (empty table, bad shapes), AF_EPRECISION (dtype),
 * AF_EALIAS (two targets overlap). */
int af_table_create(const af_segment_desc* segments, int32_t n_segments, int32_t target_dtype,
                    int32_t factor_dtype, af_table** out);
int af_table_destroy(af_table* table);
/* n_units: persistent-kernel work units; fast_path bits: 1 = TMA kernels apply, 2 = tensor path
 * (mma.sync) applies, 4 = the tcgen05 / TMEM kernels apply and are enabled (af_set_umma). */
int af_table_info(const af_table* table, int32_t* n_segments, int64_t* target_elems,
                  int32_t* n_units, int32_t* fast_path);
/* Device-side validation result of the launches issued on `stream` so far (SYNCHRONISES the
 * stream): 0, or the AF_E* code a kernel raised because a device-resident decision named an
 * expert outside the bank (adapters.py:199-200) or carried more than max_k experts; the
 * offending launch touched nothing.  Reading clears the flag. */
int af_table_status(af_table* table, void* stream);
/* Asynchronous form of the same check, for callers that already read something back every step
 * (model.py:396: the next token): the table's kernels raise into `word_dev` -- a caller-owned,
 * zero-initialised int32 in device memory (NULL: back to the table's own word) -- so that ONE
 * device-to-host copy returns the step's result and its status together.  The word is sticky
 * until the caller clears it; af_flag_message names a raised code.  Codes: AF_EINDEX / AF_EVALUE
 * (unusable device decision, adapters.py:199-200), AF_ECUDA (a chained launch gave up at a phase
 * barrier), AF_ESTATE (KV cache full). */
int af_table_set_error_word(af_table* table, int32_t* word_dev);
const char* af_flag_message(int32_t flag);

/* ---- pre-gating router --------------------------------------------------------------
 * Replaces: routing.py:49-78 `route` / routing.py:81-89 `pre_gate`, fused with the row
 * gather of model.py:248-258 `_embed_token` when `token_dev` is given.
 *   router_w : N x d (bf16 or f32), row-major, read-only
 *   x        : d-vector (x_dtype); if token_dev != NULL, x is the embedding TABLE and the
 *              routed vector is row *token_dev of it (token range is the caller's check)
 *   out_dev  : af_decision in device memory (consumed by af_fused_switch without a host
 *              round trip); logits_dev optional N floats
 * Errors: AF_EVALUE when k is outside [1, min(N, AF_MAX_K)] (routing.py:57-58). */
int af_pregate(const void* router_w, int32_t w_dtype, int32_t n_experts, int32_t d, const void* x,
               int32_t x_dtype, const int32_t* token_dev, int32_t k, af_decision* out_dev,
               float* logits_dev, void* stream);

/* ---- fused switch -------------------------------------------------------------------
 * Replaces: per token, adapters.py:188-211 `concat_gated` x L, adapters.py:214-233
 * `build_switch` x L and adapters.py:236-258 `merge_all` -> linalg.py:306-346 `sgmm`
 * (model.py:350-357): ONE persistent launch over every segment of the table.
 *   prev_dev / cur_dev : device decisions; NULL = empty concat (first token / final
 *                        unmerge, adapters.py:150-156).
 *   prev_host/cur_host : alternative host copies (used when the *_dev pointer is NULL
 *                        and the host pointer is not).
 *   max_k              : upper bound of k in the device decisions (the model's top_k); sizes the
 *                        launch.  Ignored for host decisions.
 *   scale              : LoRA scale folded into every gate (the reference fixes it to 1,
 *                        SPEC.md:197).
 * `af_merge` == switch with empty prev; `af_unmerge` == switch with empty cur
 * (merge_all(sign=-1), adapters.py:236-258; model.py:460-474 `finalize_generation`).
 * Errors: AF_EVALUE (bad mode/compute), AF_ESTATE (FROM_PRISTINE without pristine),
 * AF_EINDEX (host decision names an expert outside the bank). */
int af_fused_switch(af_table* table, const af_decision* prev_dev, const af_decision* cur_dev,
                    const af_decision* prev_host, const af_decision* cur_host, int32_t max_k,
                    float scale, int32_t mode, int32_t compute, void* stream);
int af_merge(af_table* table, const af_decision* dec_dev, const af_decision* dec_host, int32_t max_k,
             float scale, int32_t compute, void* stream);
int af_unmerge(af_table* table, const af_decision* dec_dev, const af_decision* dec_host,
               int32_t max_k, float scale, int32_t compute, void* stream);

/* linalg.py:306-346 `sgmm` on a table of MATERIALISED segments: target += sign * up @ down
 * for every segment in one launch.  Errors: AF_EVALUE when sign is not +1/-1. */
int af_sgmm(af_table* table, int32_t sign, int32_t compute, void* stream);

/* model.py:308-312 `_refresh_from_pristine`: live <- pristine for every segment. */
int af_refresh_from_pristine(af_table* table, void* stream);
/* model.py:231-236 `max_backbone_deviation`: max |live - pristine| -> *out_dev (f32). */
int af_max_deviation(af_table* table, float* out_dev, void* stream);

/* ---- bs=1 decode kernels ------------------------------------------------------------
 * af_gemv  : y = W x, W rows x cols (bf16/f32).  Replaces linalg.py:246-259 `gemm` used as
 *            the backbone GEMV (model.py:288) with the epilogue of model.py:298-305 fused.
 *            x and res are f32 vectors; out is f32.  out must not alias x.
 * af_gemv_t: y = W^T x, W rows x cols, x has `rows` entries, y has `cols`.  Replaces
 *            model.py:261-263 `_unembed` (x^T (1 x d) @ unembed (d x V)).
 * af_argmax: lowest index of the maximum (model.py:396 `np.argmax`). */
int af_gemv(const void* w, int32_t w_dtype, int32_t rows, int32_t cols, int64_t ld, const float* x,
            float* out, int32_t epilogue, const float* res, void* stream);
int af_gemv_t(const void* w, int32_t w_dtype, int32_t rows, int32_t cols, int64_t ld, const float* x,
              float* out, void* stream);
int af_argmax(const float* v, int32_t n, int32_t* out_dev, void* stream);
/* model.py:248-258 `_embed_token`: out[0:d] = (f32) table[*token_dev][0:d]. */
int af_embed(const void* table, int32_t dtype, int32_t d, const int32_t* token_dev, float* out,
             void* stream);

/* ---- Llama-shaped block, bs=1 (BASELINE.json configs 2-5) ----------------------------
 * The reference's layer is x + gelu(W x) (model.py:266-305); the metric's configurations are
 * Llama-shaped, for which the reference has no dataflow.  These are the
 * merged-path forward of model.py:367-371 for that block: plain GEMVs over the live weights
 * with the small ops fused in.
 *
 * af_gemv_fused : out = epilogue(W . prologue(x)); W rows x cols bf16 (cols % 8 == 0).
 *    prologue AF_PRO_RMSNORM : x * rsqrt(mean(x^2) + eps) * norm_w        (x has cols entries)
 *    prologue AF_PRO_SILU_MUL: silu(x[c]) * x[cols + c]                   (x has 2*cols entries)
 *    epilogue as af_gemv.
 * af_attn_decode: RoPE(q, k) at position *pos_dev, append k/v to the bf16 cache, single-query
 *    GQA attention over positions 0..*pos_dev.  qkv = [q | k | v] f32, caches
 *    [n_kv][max_seq][head_dim] bf16, cos/sin [max_seq][head_dim/2] f32.  n_split > 1 spreads
 *    the positions of each head over n_split CTAs (long contexts); it needs a workspace of
 *    n_heads * n_split * (head_dim + 2) floats and n_heads zero-initialised int32 tickets.
 * af_argmax_val : argmax + the winning value, index shifted by index_offset (vocab-parallel
 *    lm_head).
 * af_step_advance: end-of-step bookkeeping in one launch so a decode step is a static CUDA
 *    graph: prev <- cur decision, *pos += 1, *step += 1, history[step] = *next,
 *    *token = forced ? forced[(step+1) % n_forced] : *next.  Any pointer may be NULL. */
#define AF_PRO_NONE 0
#define AF_PRO_RMSNORM 1
#define AF_PRO_SILU_MUL 2
#define AF_PRO_RMSNORM_DEFERRED 3 /* af_switch_gemv_chain on the tcgen05 path only: x' = x * norm_w; the scale
                                     rsqrt(mean(x^2) + eps) is written to inv_out by one CTA and applied by the
                                     consumer of the phase's outputs (inv_in / qkv_scale_dev) */
int af_gemv_fused(const void* w, int32_t rows, int32_t cols, int64_t ld, const float* x, float* out,
                  int32_t prologue, const float* norm_w, float eps, int32_t epilogue, const float* res,
                  void* stream);
/* af_gemv_chain : up to four af_gemv_fused calls whose inputs depend on each other's outputs
 *    (o -> gate|up -> down -> next layer's q|k|v, or -> lm_head) as ONE persistent launch.  The
 *    weights of every phase stream through one shared-memory ring without stopping at a phase
 *    boundary; only the consumers wait there (phase_done_dev: n_phases - 1 int32 counters, zeroed by
 *    the caller).  Same arithmetic contract as af_gemv_fused per phase; a row is summed by one warp
 *    in a fixed order.  The launch is one CTA per SM, all co-resident; a CTA that waits ~2 s at a
 *    phase barrier raises AF_ECUDA in *err_flag_dev (may be NULL) and every CTA stops waiting, so a
 *    lost CTA ends the launch with an error instead of a hang or silently wrong outputs. */
typedef struct af_gv_phase {
    const void* w;       /* rows x cols bf16, row pitch ld                                  */
    int32_t rows, cols;
    int64_t ld;
    const float* x;      /* cols entries (2 * cols for AF_PRO_SILU_MUL)                      */
    float* out;          /* rows entries                                                     */
    const float* res;    /* epilogue residual or NULL                                        */
    const float* norm_w; /* RMSNorm weight or NULL                                           */
    float eps;
    int32_t prologue, epilogue;
} af_gv_phase;
int af_gemv_chain(const af_gv_phase* phases, int32_t n_phases, int32_t* phase_done_dev,
                  int32_t* err_flag_dev, int32_t pdl, void* stream);
/* af_forward_persistent : the whole merged-path forward of one token (model.py:367-371 on the Llama block) as ONE
 *    persistent launch driven by a device-side phase table: q|k|v(0), then per layer attention (two phases: partials
 *    per (head, 64-position chunk), combine), o, gate|up, down and the next layer's q|k|v (the lm_head after the last
 *    layer).  GEMV phases (kind AF_FW_GEMV) follow af_gemv_chain's contract; AF_FW_ATTN_PARTIAL reads q|k|v of the new
 *    token from `x` (f32, [n_heads*hd | n_kv*hd | n_kv*hd]), applies RoPE at *pos_dev, appends k / v to this layer's
 *    bf16 caches and writes per-chunk softmax partials to `workspace` (n_heads * ceil(max_seq / 64) * (head_dim + 2)
 *    floats); AF_FW_ATTN_COMBINE writes the n_heads * head_dim attention outputs to `out`.  head_dim 64 or 128.
 *    The table lives in DEVICE memory (phases_dev) and is validated from its host copy by af_forward_validate, which
 *    also returns the shared-memory vector length the launch needs (max_cols).  phase_done_dev: n_phases int32
 *    counters zeroed by the caller; err_flag_dev as in af_gemv_chain. */
#define AF_FW_GEMV 0
#define AF_FW_ATTN_PARTIAL 1
#define AF_FW_ATTN_COMBINE 2
typedef struct af_fw_phase {
    const void* w;
    const float* x;
    float* out;
    const float* res;
    const float* norm_w;
    void* k_cache;
    void* v_cache;
    int64_t ld;
    int32_t rows, cols;
    float eps;
    int32_t prologue, epilogue, kind;
} af_fw_phase;
int af_forward_validate(const af_fw_phase* phases_host, int32_t n_phases, int32_t n_heads, int32_t n_kv_heads,
                        int32_t head_dim, int32_t* max_cols_out);
int af_forward_persistent(const af_fw_phase* phases_dev, int32_t n_phases, int32_t max_cols, const float* cos_table,
                          const float* sin_table, const int32_t* pos_dev, int32_t n_heads, int32_t n_kv_heads,
                          int32_t head_dim, int32_t max_seq, float* workspace, int32_t* phase_done_dev,
                          int32_t* err_flag_dev, int32_t pdl, void* stream);
int af_attn_decode(const float* qkv, void* k_cache, void* v_cache, const float* cos_table,
                   const float* sin_table, const int32_t* pos_dev, int32_t n_heads, int32_t n_kv_heads,
                   int32_t head_dim, int32_t max_seq, int32_t n_split, float* workspace,
                   int32_t* tickets, float* out, void* stream);
int af_argmax_val(const float* v, int32_t n, int32_t index_offset, int32_t* out_idx_dev,
                  float* out_val_dev, void* stream);
int af_step_advance(af_decision* prev_dev, const af_decision* cur_dev, int32_t* pos_dev,
                    int32_t* step_dev, int32_t* token_dev, const int32_t* next_dev,
                    const int32_t* forced_dev, int32_t n_forced, int32_t* history_dev,
                    int32_t n_history, void* stream);

/* ---- fused switch + GEMV ("chase" mode) -------------------------------
 * The steady decode step moves every weight twice for the switch (read + write) and once more
 * for the forward GEMV.  These entry points remove the third pass: a projection's segments are
 * switched (adapters.py:236-258 -> linalg.py:306-346) and, while each freshly merged and rounded
 * tile is still in registers, multiplied with the projection's input vector (model.py:288).
 * One launch per projection of the Llama block (q|k|v, o, gate|up, down); a token costs
 * 2 x W bytes instead of 3 x W.
 *
 * af_group_create : segments of `table` that share one input vector, in the order their outputs
 *    are concatenated; builds an evenly split tile schedule for one launch.
 * af_switch_gemv  : W <- W + delta(cur) - delta(prev) on the group's segments AND
 *    acc_out[row] += fix(W_new[row] . x).  prev_dev / cur_dev / max_k / scale / mode as
 *    af_fused_switch (both NULL: no switch, the launch is a plain GEMV over the live weights).
 *    Input vector:  h = (res ? res : 0) + (acc_in ? fix^-1(acc_in) : xin);  x = prologue(h)
 *    (AF_PRO_NONE / AF_PRO_RMSNORM with norm_w, eps / AF_PRO_SILU_MUL over [gate | up], no res).
 *    h_out (optional) receives h -- the residual stream -- written by one CTA.
 *    acc_out: y_rows 64-bit fixed-point accumulators (value * 2^AF_FIX_SHIFT), ZEROED BY THE CALLER
 *    before the launch; the per-strip partial dot products are added with integer atomics, so the
 *    result does not depend on CTA arrival order (deterministic).
 *    pdl != 0: launched with programmatic stream serialization -- the launch streams its weights
 *    while the previous kernel of the stream drains; the previous kernel must be one of this
 *    library's decode kernels (they all execute griddepcontrol.wait).
 * af_accum_to_f32 : out = (res ? res : 0) + fix^-1(acc)   (hand-over to af_gemv_fused / lm_head).
 * af_attn_decode_fix : af_attn_decode reading q|k|v from fixed-point accumulators, times
 *    *qkv_scale_dev when given (the deferred RMSNorm scale of the launch that produced them).
 *
 * Chains: up to 4 projections whose inputs depend on each other's outputs (o -> gate|up -> down ->
 * next layer's q|k|v) run in ONE launch (af_chain_create / af_switch_gemv_chain).  The weight
 * stream never stops at a phase boundary -- the tiles of the next projection fill the
 * shared-memory ring meanwhile; only the consumers wait, on a device counter every CTA bumps when
 * its partial sums of the phase are out.  phase_done_dev: n_phases - 1 int32 counters, zeroed by
 * the caller before the launch.  All CTAs of the launch must be co-resident (grid <= SM count, one
 * CTA per SM; the library sizes it so); a lost CTA raises AF_ECUDA on the table after ~2 s instead
 * of hanging. */
#define AF_FIX_SHIFT 40
typedef struct af_group af_group;
typedef struct af_gemv_phase {
    const float* xin;       /* plain input vector, or NULL when acc_in is given                    */
    const int64_t* acc_in;  /* fixed-point output of an earlier launch / phase                     */
    const float* res;       /* optional residual added to the input                                */
    float* h_out;           /* optional: receives h = res + input (the residual stream)            */
    const float* norm_w;    /* RMSNorm weight (AF_PRO_RMSNORM)                                     */
    int64_t* acc_out;       /* y_rows accumulators of this phase, zeroed by the caller             */
    float eps;
    int32_t prologue;
    float* inv_out;         /* AF_PRO_RMSNORM_DEFERRED: receives the scale of this phase's input   */
    const float* inv_in;    /* scale of this phase's input accumulators (deferred by their producer) */
} af_gemv_phase;
int af_group_create(af_table* table, const int32_t* seg_ids, int32_t n, af_group** out);
/* seg_ids: the phases' segment lists back to back; phase_len[p] segments belong to phase p. */
int af_chain_create(af_table* table, const int32_t* seg_ids, const int32_t* phase_len, int32_t n_phases,
                    af_group** out);
/* af_chain_create with a measured work split: cta_share[ph * n_cta + c] > 0 is the relative share of phase ph's
 * tiles CTA c gets (NULL = equal shares).  Every CTA of a chained launch meets the others at each phase barrier,
 * so the slowest SM sets the pace; SM rates differ by a few per cent with their position on the chip, identically
 * in every launch, and a caller that has timed them (af_set_timeline) can hand the split back.  The schedule
 * changes which CTA takes which tile and nothing else: weights and accumulators are bit-identical. */
int af_chain_create_weighted(af_table* table, const int32_t* seg_ids, const int32_t* phase_len, int32_t n_phases,
                             const float* cta_share, int32_t n_cta, af_group** out);
int af_group_destroy(af_group* group);
/* x_len / y_rows: arrays of n_phases entries (4 is always enough).  grid: CTAs of a launch over the group (the
 * tcgen05 schedule's when the table is on that path; what a peer counter is compared against, times n_peers). */
int af_group_info(const af_group* group, int32_t* n_phases, int32_t* x_len, int32_t* y_rows, int32_t* n_units,
                  int32_t* grid, int64_t* tiles);
/* flags of af_switch_gemv_chain (af_switch_gemv takes AF_CHAIN_PDL as its `pdl` argument) */
#define AF_CHAIN_PDL 1           /* programmatic stream serialization, see af_switch_gemv          */
#define AF_CHAIN_PLAN_PREBUILT 2 /* the block list of (prev, cur, scale, mode) was built by          */
                                 /* af_plan_build earlier on this stream: skip the per-launch build */
int af_switch_gemv_chain(af_group* group, const af_decision* prev_dev, const af_decision* cur_dev,
                         int32_t max_k, float scale, int32_t mode, const af_gemv_phase* phases,
                         int32_t n_phases, int32_t* phase_done_dev, int32_t flags, void* stream);
/* ---- tensor parallelism without a collective between the launches ----------------------------
 * No reference counterpart (the reference is single-process; BASELINE configs[3..4] name TP 2 / 4 / 8).
 * Every rank maps one buffer holding the fixed-point accumulators and phase counters of every other rank
 * (NVLink peer memory: torch symmetric memory or CUDA IPC handles on the host side, `llama.PeerBuffer`) at own address + peer_offset_bytes[w];
 * the list includes the rank itself (offset 0) and has the same ORDER on every rank only by convention -- the
 * kernels never use the index.  af_group_set_peers marks the row-parallel phases of a chain (bit ph of
 * reduce_phase_mask: o and down): a marked phase adds its partial sums into EVERY rank's acc_out with system-scope
 * integer atomics (exact in any order -- the all-reduce is part of the GEMV epilogue) and is reported on every
 * rank's phase counter, so the next phase starts on the reduced vector once grid * n_peers CTAs have reported.
 * Requirements: tcgen05 path; identical chain shapes (hence grids) on all ranks; acc_out of the marked phases and
 * phase_done_dev inside the mapped buffer; phase_done_dev then holds n_phases counters when the LAST phase is
 * marked (its consumer is a later launch: af_peer_wait on counter n_phases - 1 for grid * n_peers).
 * n_peers == 0 clears the setting.  Errors: AF_EVALUE, AF_EDIM (alignment), AF_EALIAS, AF_ESTATE (not tcgen05). */
int af_group_set_peers(af_group* group, int32_t n_peers, const int64_t* peer_offset_bytes, int32_t reduce_phase_mask);
/* Once per token, after this rank has zeroed its accumulators / counters and before any rank may push into them:
 * bumps counter_dev on every rank (a monotonic count, never reset) and waits until all n_peers ranks have bumped
 * this rank's; *epoch_dev (device-resident, zero-initialised, private to the rank) counts the barriers so far. */
int af_peer_barrier(int32_t* counter_dev, int32_t* epoch_dev, int32_t n_peers, const int64_t* peer_offset_bytes,
                    int32_t* err_flag_dev, void* stream);
/* The two exchanges of a tensor-parallel token that are not sums, over the same peer mappings, so that a step holds no
 * library collective (and captures as a CUDA graph without one):
 * af_peer_bcast  -- rank 0's decision record (`llama.Collectives.broadcast_decision`; SURVEY.md 8b `af_bcast_decision`):
 *    the root (is_root != 0) copies `bytes` from src_dev into slot_dev of EVERY rank and bumps every rank's counter; each
 *    rank waits until its counter has reached its own number of broadcasts so far (*epoch_dev) and copies its slot to dst_dev.
 * af_peer_argmax -- the vocab-parallel argmax (model.py:396 over the ranks' lm_head slices): every rank writes its
 *    (value, index) pair into slot my_slot of every rank's slots_dev (n_peers 8-byte words), bumps every rank's counter,
 *    waits for the n pairs of this round and writes the index of the largest value (lowest index on ties) to out_idx_dev.
 * slot_dev / slots_dev / counter_dev live in the mapped buffer, each call kind with its own counter and epoch word. */
int af_peer_bcast(const void* src_dev, void* slot_dev, void* dst_dev, int32_t bytes, int32_t is_root, int32_t* counter_dev,
                  int32_t* epoch_dev, int32_t n_peers, const int64_t* peer_offset_bytes, int32_t* err_flag_dev, void* stream);
int af_peer_argmax(const float* val_dev, const int32_t* idx_dev, void* slots_dev, int32_t my_slot, int32_t* counter_dev,
                   int32_t* epoch_dev, int32_t n_peers, const int64_t* peer_offset_bytes, int32_t* out_idx_dev,
                   int32_t* err_flag_dev, void* stream);
/* Stream-ordered wait until *counter_dev >= target (system-scope acquire); ~2 s -> AF_ECUDA in *err_flag_dev.  Every
 * cross-rank wait of the library (this one, af_peer_barrier / _bcast / _argmax, the phase barriers of a launch with
 * peers) gives up after ~2 ms once *err_flag_dev is already non-zero: a dead rank fails the step in seconds. */
int af_peer_wait(const int32_t* counter_dev, int32_t target, int32_t* err_flag_dev, void* stream);
/* adapters.py:188-233 (`concat_gated` + `build_switch` bookkeeping) once per token: turns the two
 * device decisions into the table's block list (experts present on both sides collapse to one block
 * of weight g_new - g_old).  The launches of the token that pass AF_CHAIN_PLAN_PREBUILT read it
 * instead of rebuilding it; validation errors surface through af_table_status as usual. */
int af_plan_build(af_table* table, const af_decision* prev_dev, const af_decision* cur_dev, int32_t max_k,
                  float scale, int32_t mode, void* stream);
int af_switch_gemv(af_group* group, const af_decision* prev_dev, const af_decision* cur_dev, int32_t max_k,
                   float scale, int32_t mode, const float* xin, const int64_t* acc_in, const float* res,
                   float* h_out, int32_t prologue, const float* norm_w, float eps, int64_t* acc_out,
                   int32_t pdl, void* stream);
/* Profiling aid: the next n_launches af_switch_gemv[_chain] launches each write per-CTA
 * %globaltimer stamps (grid x AF_TIMELINE_SLOTS uint64: entry, plan ready, first slab, pdl wait
 * passed, first/last W load issued, storer done, consumers done, then per phase: wait begins,
 * barrier passed, prologue done, first tile computed; then %smid) to buffer_dev + i * stride_elems.
 * buffer_dev == NULL turns the probe off. */
#define AF_TIMELINE_SLOTS 42
int af_set_timeline(uint64_t* buffer_dev, int32_t n_launches, int64_t stride_elems);
int af_accum_to_f32(const int64_t* acc, const float* res, float* out, int32_t n, void* stream);
int af_attn_decode_fix(const int64_t* qkv_fix, const float* qkv_scale_dev, void* k_cache, void* v_cache,
                       const float* cos_table, const float* sin_table, const int32_t* pos_dev, int32_t n_heads,
                       int32_t n_kv_heads, int32_t head_dim, int32_t max_seq, int32_t n_split, float* workspace,
                       int32_t* tickets, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ADAFUSE_B200_H */
