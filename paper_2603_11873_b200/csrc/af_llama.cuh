// af_llama.cuh -- bs=1 decode kernels of the Llama-shaped block (BASELINE.json configs 2-5).
//
// The reference's decoder is `x + gelu(W x)` per layer (model.py:266-305); the configurations
// the metric is quoted on are Llama-shaped (q/k/v/o/gate/up/down, GQA), for which the
// reference has no dataflow.  These kernels are the merged-path forward of
// model.py:367-371 for that block: after the fused switch every projection is a PLAIN GEMV
// over the live bf16 weights.  All of them are HBM-bound streaming reads of W; everything
// small (RMSNorm, SiLU*up, residual adds, RoPE, the KV append) is fused into a GEMV
// prologue/epilogue or the attention kernel so a layer is 5 launches.
#pragma once

#include "af_common.cuh"

namespace af {

constexpr int kPrologueNone = 0;
constexpr int kPrologueRmsNorm = 1;   // xs = x * rsqrt(mean(x^2) + eps) * norm_w
constexpr int kPrologueSiluMul = 2;   // xs = silu(x[c]) * x[cols + c]   (x holds [gate | up])

#ifndef AF_GEMV_RB
#define AF_GEMV_RB 4
#endif
#ifndef AF_GEMV_MINB
#define AF_GEMV_MINB 4   /* 64 registers -> 4 CTAs (32 warps) per SM: measured best, profiles/r01_sweep_gemv.txt */
#endif
#ifndef AF_GEMV_THREADS
#define AF_GEMV_THREADS 256
#endif
constexpr int kGemvFThreads = AF_GEMV_THREADS;
constexpr int kGemvRB = AF_GEMV_RB;           // rows per batch (one partial sum each per thread)
constexpr int kGemvPass = kGemvFThreads * 8;  // columns covered by the CTA per pass (16 B per thread)

__device__ __forceinline__ void unpack8(const uint4 v, float (&f)[8]) {
    f[0] = bf16lo_to_f32(v.x); f[1] = bf16hi_to_f32(v.x); f[2] = bf16lo_to_f32(v.y); f[3] = bf16hi_to_f32(v.y);
    f[4] = bf16lo_to_f32(v.z); f[5] = bf16hi_to_f32(v.z); f[6] = bf16lo_to_f32(v.w); f[7] = bf16hi_to_f32(v.w);
}

// Streaming 16-byte load that does not pollute L1 (W is read exactly once per token).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
#ifdef AF_GEMV_L2_256
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
#else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
#endif
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}


// 1-D bulk copy global -> shared, completing on an mbarrier (UBLKCP); 16-byte aligned, size % 16 == 0.
__device__ __forceinline__ void gv_bulk_load(uint32_t smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// y = epilogue(W . prologue(x)), W rows x cols bf16 row-major (cols % 8 == 0, 16-byte aligned rows).
//
// HBM-bound streaming read of W, one persistent CTA per SM, rows split EVENLY over the grid so
// every SM streams the same number of bytes.  W never goes through registers on its way in: a
// producer thread streams it with 1-D bulk copies (TMA engine) into a ring of kGvStage-byte
// stages guarded by full/empty mbarriers -- up to `n_stages` x 16 KB per SM are in flight no
// matter what the consumer warps are doing.  The producer starts BEFORE the prologue and before
// pdl_wait(): under programmatic dependent launch the ring is already full of this kernel's
// weights while the previous kernel drains and while the consumers build xs (RMSNorm / SiLU*up).
//
// A stage holds one kGvCH-column chunk of 8 consecutive rows, one row per consumer warp: a warp
// accumulates its own row across the chunks and finishes with a shuffle reduction, so the
// steady state has no block-wide barrier at all.
constexpr int kGvWarps = 8;                       // consumer warps = rows per group
constexpr int kGvMaxStages = 10;
constexpr int kGvMaxProd = 4;

// CH = columns per row chunk (one bulk copy of CH*2 bytes), NPROD = producer threads (one per
// warp; a single thread can issue a bulk copy only every ~80-100 cycles, so 8 copies of 2 KB per
// 16 KB stage would cap one SM below its share of HBM bandwidth).
template <int CH, int NPROD>
__global__ void __launch_bounds__(kGvWarps * 32 + 32 * NPROD, 1)
gemv_tma_kernel(const __nv_bfloat16* __restrict__ w, int rows, int cols, long long ld, const float* __restrict__ x,
                float* __restrict__ out, int prologue, const float* __restrict__ norm_w, float eps, int epilogue,
                const float* __restrict__ res, int n_stages) {
    constexpr int kStage = kGvWarps * CH * 2;
    extern __shared__ __align__(128) unsigned char gv_smem[];
    // layout: [stages x kStage] [xs: cols f32] ; barriers static
    __shared__ uint64_t full[kGvMaxStages], empty[kGvMaxStages];
    __shared__ float redn[kGvWarps];
    float* xs = reinterpret_cast<float*>(gv_smem + (size_t)n_stages * kStage);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_launch_dependents();
    const int r_begin = (int)((long long)rows * blockIdx.x / gridDim.x);
    const int r_end = (int)((long long)rows * (blockIdx.x + 1) / gridDim.x);
    const int n_groups = (r_end - r_begin + kGvWarps - 1) / kGvWarps;
    const int n_ch = (cols + CH - 1) / CH;
    const int total = n_groups * n_ch;
    if (tid == 0) {
        for (int s = 0; s < n_stages; ++s) {
            mbar_init(&full[s], NPROD);
            mbar_init(&empty[s], kGvWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp >= kGvWarps) {
        // ===================== producers: stream W, independent of the previous kernel =====================
        if (lane == 0) {
            const int who = warp - kGvWarps;
            const uint32_t base = smem_u32(gv_smem);
            for (int it = 0; it < total; ++it) {
                const int stage = it % n_stages;
                const uint32_t ph = (it / n_stages) & 1;
                const int g = it / n_ch, ch = it % n_ch;
                const int row0 = r_begin + g * kGvWarps;
                const int nrow = min(kGvWarps, r_end - row0);
                const int c0 = ch * CH;
                const uint32_t bytes = (uint32_t)min(CH, cols - c0) * 2;
                int mine = 0;
                for (int r = who; r < nrow; r += NPROD) ++mine;
                mbar_wait(&empty[stage], ph ^ 1);
                mbar_expect_tx(&full[stage], bytes * mine);
                for (int r = who; r < nrow; r += NPROD)
                    gv_bulk_load(base + stage * kStage + r * (CH * 2), w + (long long)(row0 + r) * ld + c0, bytes, &full[stage]);
            }
        }
        return;
    }

    // ===================== consumers =====================
    pdl_wait();  // x / res come from the previous kernel
    constexpr int kC = kGvWarps * 32;
    if (prologue == kPrologueRmsNorm) {
        float ss = 0.f;
        for (int c = tid * 4; c < cols; c += kC * 4) {
            const float4 v = *reinterpret_cast<const float4*>(x + c);
            *reinterpret_cast<float4*>(xs + c) = v;
            ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
        }
        ss = warp_sum(ss);
        if (lane == 0) redn[warp] = ss;
        named_bar_sync(1, kC);
        float tot = 0.f;
#pragma unroll
        for (int i = 0; i < kGvWarps; ++i) tot += redn[i];
        const float inv = rsqrtf(tot / (float)cols + eps);
        for (int c = tid * 4; c < cols; c += kC * 4) {
            float4 v = *reinterpret_cast<float4*>(xs + c);
            const float4 nw = *reinterpret_cast<const float4*>(norm_w + c);
            v.x *= inv * nw.x; v.y *= inv * nw.y; v.z *= inv * nw.z; v.w *= inv * nw.w;
            *reinterpret_cast<float4*>(xs + c) = v;
        }
    } else if (prologue == kPrologueSiluMul) {
        for (int c = tid * 4; c < cols; c += kC * 4) {
            const float4 g = *reinterpret_cast<const float4*>(x + c);
            const float4 u = *reinterpret_cast<const float4*>(x + cols + c);
            float4 v;
            v.x = g.x / (1.0f + expf(-g.x)) * u.x;
            v.y = g.y / (1.0f + expf(-g.y)) * u.y;
            v.z = g.z / (1.0f + expf(-g.z)) * u.z;
            v.w = g.w / (1.0f + expf(-g.w)) * u.w;
            *reinterpret_cast<float4*>(xs + c) = v;
        }
    } else {
        for (int c = tid * 4; c < cols; c += kC * 4) *reinterpret_cast<float4*>(xs + c) = *reinterpret_cast<const float4*>(x + c);
    }
    named_bar_sync(1, kC);

    float acc0 = 0.f, acc1 = 0.f;
    for (int it = 0; it < total; ++it) {
        const int stage = it % n_stages;
        const uint32_t ph = (it / n_stages) & 1;
        const int g = it / n_ch, ch = it % n_ch;
        const int row = r_begin + g * kGvWarps + warp;
        const int c0 = ch * CH;
        const int width = min(CH, cols - c0);
        mbar_wait(&full[stage], ph);
        if (row < r_end) {
            const unsigned char* wrow = gv_smem + (size_t)stage * kStage + warp * (CH * 2);
#pragma unroll
            for (int i = 0; i < CH / 256; ++i) {
                const int c = lane * 8 + i * 256;
                if (c < width) {
                    const uint4 v = *reinterpret_cast<const uint4*>(wrow + c * 2);
                    const float4 xa = *reinterpret_cast<const float4*>(xs + c0 + c);
                    const float4 xb = *reinterpret_cast<const float4*>(xs + c0 + c + 4);
                    float wf[8];
                    unpack8(v, wf);
                    acc0 = fmaf(wf[0], xa.x, acc0); acc1 = fmaf(wf[1], xa.y, acc1); acc0 = fmaf(wf[2], xa.z, acc0); acc1 = fmaf(wf[3], xa.w, acc1);
                    acc0 = fmaf(wf[4], xb.x, acc0); acc1 = fmaf(wf[5], xb.y, acc1); acc0 = fmaf(wf[6], xb.z, acc0); acc1 = fmaf(wf[7], xb.w, acc1);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (ch == n_ch - 1) {
            const float y = warp_sum(acc0 + acc1);
            acc0 = acc1 = 0.f;
            if (lane == 0 && row < r_end) {
                float o = y;
                if (epilogue == AF_EPI_GELU_RESIDUAL)
                    o = res[row] + 0.5f * y * (1.0f + erff(y * 0.70710678118654752440f));
                else if (epilogue == AF_EPI_RESIDUAL)
                    o = res[row] + y;
                out[row] = o;
            }
        }
    }
}

// ---- register-streamed variant (no shared-memory ring for W): kept selectable (af_set_gemv_variant)
//      so the two streaming strategies can be measured against each other on the same launch chain ----
// y = epilogue(W . prologue(x)), W rows x cols bf16 row-major (cols % 8 == 0, 16-byte aligned rows).
//
// HBM-bound streaming read of W.  Rows are split EVENLY over the grid (grid = SMs x resident
// CTAs, so every SM streams the same number of bytes); inside a CTA all 256 threads cooperate
// on a batch of kGemvRB rows: thread t owns the 16-byte chunk t of every 4 KB pass of a row.
// The loop is software-pipelined two items deep (8 independent 16-byte loads in flight per
// thread while a third item is consumed), the first loads are issued BEFORE the prologue and
// before pdl_wait(), so the prologue and the tail of the previous kernel hide under them.
__global__ void __launch_bounds__(kGemvFThreads, AF_GEMV_MINB) gemv_fused_kernel(const __nv_bfloat16* __restrict__ w, int rows, int cols,
                                                                    long long ld, const float* __restrict__ x,
                                                                    float* __restrict__ out, int prologue,
                                                                    const float* __restrict__ norm_w, float eps, int epilogue,
                                                                    const float* __restrict__ res) {
    extern __shared__ __align__(16) float xs[];
    __shared__ float red[2][kGemvFThreads / 32][kGemvRB];
    __shared__ float redn[kGemvFThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kGemvFThreads / 32;
    pdl_launch_dependents();
    const int r_begin = (int)((long long)rows * blockIdx.x / gridDim.x);
    const int r_end = (int)((long long)rows * (blockIdx.x + 1) / gridDim.x);
    const int n_pass = (cols + kGemvPass - 1) / kGemvPass;
    const int n_batch = (r_end - r_begin + kGemvRB - 1) / kGemvRB;
    const int total = n_batch * n_pass;

    auto issue = [&](int it, uint4 (&v)[kGemvRB]) {
        if (it >= total) return;
        const int b = it / n_pass, c = (it % n_pass) * kGemvPass + tid * 8;
#pragma unroll
        for (int i = 0; i < kGemvRB; ++i) {
            const int row = r_begin + b * kGemvRB + i;
            v[i] = (row < r_end && c < cols) ? ldg_stream(w + (long long)row * ld + c) : make_uint4(0u, 0u, 0u, 0u);
        }
    };
    uint4 b0[kGemvRB], b1[kGemvRB], b2[kGemvRB];
    issue(0, b0);
    issue(1, b1);

    pdl_wait();  // x / res come from the previous kernel
    if (prologue == kPrologueRmsNorm) {
        float ss = 0.f;
        for (int c = tid * 4; c < cols; c += kGemvFThreads * 4) {
            const float4 v = *reinterpret_cast<const float4*>(x + c);
            *reinterpret_cast<float4*>(xs + c) = v;
            ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
        }
        ss = warp_sum(ss);
        if (lane == 0) redn[warp] = ss;
        __syncthreads();
        float tot = 0.f;
#pragma unroll
        for (int i = 0; i < nwarps; ++i) tot += redn[i];
        const float inv = rsqrtf(tot / (float)cols + eps);
        for (int c = tid * 4; c < cols; c += kGemvFThreads * 4) {
            float4 v = *reinterpret_cast<float4*>(xs + c);
            const float4 nw = *reinterpret_cast<const float4*>(norm_w + c);
            v.x *= inv * nw.x; v.y *= inv * nw.y; v.z *= inv * nw.z; v.w *= inv * nw.w;
            *reinterpret_cast<float4*>(xs + c) = v;
        }
    } else if (prologue == kPrologueSiluMul) {
        for (int c = tid * 4; c < cols; c += kGemvFThreads * 4) {
            const float4 g = *reinterpret_cast<const float4*>(x + c);
            const float4 u = *reinterpret_cast<const float4*>(x + cols + c);
            float4 v;
            v.x = g.x / (1.0f + expf(-g.x)) * u.x;
            v.y = g.y / (1.0f + expf(-g.y)) * u.y;
            v.z = g.z / (1.0f + expf(-g.z)) * u.z;
            v.w = g.w / (1.0f + expf(-g.w)) * u.w;
            *reinterpret_cast<float4*>(xs + c) = v;
        }
    } else {
        for (int c = tid * 4; c < cols; c += kGemvFThreads * 4)
            *reinterpret_cast<float4*>(xs + c) = *reinterpret_cast<const float4*>(x + c);
    }
    __syncthreads();

    float acc[kGemvRB] = {};
    int buf = 0;
    auto consume = [&](int it, const uint4 (&v)[kGemvRB]) {
        if (it >= total) return;
        const int b = it / n_pass, ps = it % n_pass, c = ps * kGemvPass + tid * 8;
        if (c < cols) {
            const float4 xa = *reinterpret_cast<const float4*>(xs + c);
            const float4 xb = *reinterpret_cast<const float4*>(xs + c + 4);
            const float xf[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
            for (int i = 0; i < kGemvRB; ++i) {
                float wf[8];
                unpack8(v[i], wf);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i] = fmaf(wf[j], xf[j], acc[i]);
            }
        }
        if (ps == n_pass - 1) {  // the batch is complete: CTA-wide reduction and epilogue
#pragma unroll
            for (int i = 0; i < kGemvRB; ++i) {
                const float y = warp_sum(acc[i]);
                if (lane == 0) red[buf][warp][i] = y;
                acc[i] = 0.f;
            }
            __syncthreads();
            if (tid < kGemvRB) {
                const int row = r_begin + b * kGemvRB + tid;
                if (row < r_end) {
                    float y = 0.f;
#pragma unroll
                    for (int wv = 0; wv < nwarps; ++wv) y += red[buf][wv][tid];
                    float o = y;
                    if (epilogue == AF_EPI_GELU_RESIDUAL)
                        o = res[row] + 0.5f * y * (1.0f + erff(y * 0.70710678118654752440f));
                    else if (epilogue == AF_EPI_RESIDUAL)
                        o = res[row] + y;
                    out[row] = o;
                }
            }
            buf ^= 1;
        }
    };
    for (int it = 0; it < total; it += 3) {
        issue(it + 2, b2);
        consume(it, b0);
        issue(it + 3, b0);
        consume(it + 1, b1);
        issue(it + 4, b1);
        consume(it + 2, b2);
    }
}

// Single-query GQA attention for one new token, fused with RoPE and the KV-cache append.
//   qkv     : f32 [n_heads*hd | n_kv*hd | n_kv*hd]  (output of the fused q/k/v GEMV)
//   k_cache : bf16 [n_kv][max_seq][hd], v_cache likewise; position *pos_dev is written here
//   cos/sin : f32 [max_seq][hd/2] rotary tables (rotate-half convention)
//   out     : f32 [n_heads*hd]
// Grid = n_heads x n_split CTAs (flash-decoding): split sp of head h covers a contiguous range
// of the positions 0..pos; each of its 8 warps keeps 4 positions (8 vector loads) in flight and
// runs an online softmax; the CTA writes its partial (max, sum, acc[hd]) to a workspace and the
// last CTA of a head to arrive (atomic ticket) combines the splits.  The new position's own
// (rotated, bf16-rounded) k and v are used from shared memory, so no CTA reads what a sibling
// is still appending.
constexpr int kAttnThreads = 256;
constexpr int kAttnWarps = kAttnThreads / 32;
constexpr int kAttnMaxHd = 256;
constexpr int kAttnUnroll = 8;
#ifndef AF_ATTN_POS_PER_SPLIT
#define AF_ATTN_POS_PER_SPLIT 32
#endif
constexpr int kAttnPosPerSplit = AF_ATTN_POS_PER_SPLIT;   // positions below which a further KV split does not pay

template <int EL>
__device__ __forceinline__ void load_bf16_vec(const __nv_bfloat16* p, float (&f)[EL]) {
    if constexpr (EL == 2) {
        const uint32_t v = *reinterpret_cast<const uint32_t*>(p);
        f[0] = bf16lo_to_f32(v); f[1] = bf16hi_to_f32(v);
    } else if constexpr (EL == 4) {
        const uint2 v = *reinterpret_cast<const uint2*>(p);
        f[0] = bf16lo_to_f32(v.x); f[1] = bf16hi_to_f32(v.x); f[2] = bf16lo_to_f32(v.y); f[3] = bf16hi_to_f32(v.y);
    } else if constexpr (EL == 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
        f[0] = bf16lo_to_f32(v.x); f[1] = bf16hi_to_f32(v.x); f[2] = bf16lo_to_f32(v.y); f[3] = bf16hi_to_f32(v.y);
        f[4] = bf16lo_to_f32(v.z); f[5] = bf16hi_to_f32(v.z); f[6] = bf16lo_to_f32(v.w); f[7] = bf16hi_to_f32(v.w);
    } else {
#pragma unroll
        for (int j = 0; j < EL; ++j) f[j] = __bfloat162float(p[j]);
    }
}

// EL = elements of the head dimension owned by one lane (contiguous): hd == 32 * EL for the
// vector instantiations (2, 4, 8); EL == 1 is the generic one (any even hd <= 256, lane-strided).
template <int EL>
__global__ void __launch_bounds__(kAttnThreads) attn_decode_kernel(const float* __restrict__ qkv,
                                                                   const long long* __restrict__ qkv_fix,
                                                                   const float* __restrict__ qkv_scale,
                                                                   __nv_bfloat16* __restrict__ k_cache,
                                                                   __nv_bfloat16* __restrict__ v_cache,
                                                                   const float* __restrict__ cos_t,
                                                                   const float* __restrict__ sin_t,
                                                                   const int32_t* __restrict__ pos_dev, int n_heads,
                                                                   int n_kv, int hd, int max_seq, float scale, int n_split,
                                                                   float* __restrict__ ws, int* __restrict__ tickets,
                                                                   float* __restrict__ out) {
    constexpr bool VEC = EL > 1;
    constexpr int PER = VEC ? EL : kAttnMaxHd / 32;  // accumulator slots per lane
    __shared__ float q_s[kAttnMaxHd], k_s[kAttnMaxHd], v_s[kAttnMaxHd];
    __shared__ float m_s[kAttnWarps], l_s[kAttnWarps];
    __shared__ float acc_s[kAttnWarps][kAttnMaxHd];
    __shared__ int is_last;
    const int h = blockIdx.x / n_split, sp = blockIdx.x % n_split;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int group = n_heads / n_kv, kvh = h / group;
    pdl_wait();  // qkv comes from the previous kernel
    pdl_launch_dependents();  // after the wait: a dependent's pre-wait part then never runs ahead of qkv's producer
    const int pos = *pos_dev;
    if (pos < 0 || pos >= max_seq) return;   // KV cache full: touch nothing (the host side raises StateError before it gets here)
    const int n_pos = pos + 1;
    // the grid is sized for the longest context; a short one uses fewer splits (a split below ~32 positions costs
    // more in the combine than it saves), the other CTAs of the head leave here
    n_split = min(n_split, max(1, (n_pos + kAttnPosPerSplit - 1) / kAttnPosPerSplit));
    if (sp >= n_split) return;
    const int per = (n_pos + n_split - 1) / n_split;
    const int t0 = sp * per, t1 = min(n_pos, t0 + per);
    const int half = hd >> 1;
    // q/k/v of this head: f32, or the fixed-point accumulators of a fused switch + GEMV launch
    const long long oq = (long long)h * hd, ok = (long long)n_heads * hd + (long long)kvh * hd,
                    ov = (long long)(n_heads + n_kv) * hd + (long long)kvh * hd;
    // (a launch with a deferred RMSNorm leaves q|k|v unscaled: qkv_scale holds the factor)
    const float fix_scale = (qkv_scale ? *qkv_scale : 1.0f) * (1.0f / (float)(1ll << AF_FIX_SHIFT));
    auto ld = [&](long long i) { return qkv_fix ? __ll2float_rn(qkv_fix[i]) * fix_scale : qkv[i]; };
    // RoPE (rotate-half): x'[i] = x[i] c - x[i+half] s ; x'[i+half] = x[i+half] c + x[i] s
    for (int i = tid; i < half; i += kAttnThreads) {
        const float c = cos_t[(long long)pos * half + i], s = sin_t[(long long)pos * half + i];
        const float q0 = ld(oq + i), q1 = ld(oq + i + half);
        q_s[i] = q0 * c - q1 * s;
        q_s[i + half] = q1 * c + q0 * s;
        const float k0 = ld(ok + i), k1 = ld(ok + i + half);
        // the cache stores bf16: the new position uses the rounded values too, so that a later
        // token sees exactly what this one saw
        k_s[i] = __bfloat162float(__float2bfloat16_rn(k0 * c - k1 * s));
        k_s[i + half] = __bfloat162float(__float2bfloat16_rn(k1 * c + k0 * s));
    }
    for (int i = tid; i < hd; i += kAttnThreads) v_s[i] = __bfloat162float(__float2bfloat16_rn(ld(ov + i)));
    __syncthreads();
    if (h % group == 0 && pos >= t0 && pos < t1) {  // one CTA per kv head appends to the cache
        __nv_bfloat16* kc = k_cache + ((long long)kvh * max_seq + pos) * hd;
        __nv_bfloat16* vc = v_cache + ((long long)kvh * max_seq + pos) * hd;
        for (int i = tid; i < hd; i += kAttnThreads) {
            kc[i] = __float2bfloat16_rn(k_s[i]);
            vc[i] = __float2bfloat16_rn(v_s[i]);
        }
    }
    // element e of this lane's slot j
    auto elem = [&](int j) { return VEC ? lane * EL + j : lane + 32 * j; };
    float qr[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) qr[j] = elem(j) < hd ? q_s[elem(j)] : 0.f;
    float acc[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) acc[j] = 0.f;
    float m = -INFINITY, l = 0.f;
    const __nv_bfloat16* kbase = k_cache + (long long)kvh * max_seq * hd;
    const __nv_bfloat16* vbase = v_cache + (long long)kvh * max_seq * hd;
    for (int tb = t0 + warp; tb < t1; tb += kAttnWarps * kAttnUnroll) {
        float kf[kAttnUnroll][PER], vf[kAttnUnroll][PER];
#pragma unroll
        for (int u = 0; u < kAttnUnroll; ++u) {
            const int t = tb + u * kAttnWarps;
            if (t < t1 && t != pos) {
                if constexpr (VEC) {
                    load_bf16_vec<EL>(kbase + (long long)t * hd + lane * EL, kf[u]);
                    load_bf16_vec<EL>(vbase + (long long)t * hd + lane * EL, vf[u]);
                } else {
#pragma unroll
                    for (int j = 0; j < PER; ++j) {
                        const int e = lane + 32 * j;
                        kf[u][j] = e < hd ? __bfloat162float(kbase[(long long)t * hd + e]) : 0.f;
                        vf[u][j] = e < hd ? __bfloat162float(vbase[(long long)t * hd + e]) : 0.f;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    const bool ok = t == pos && elem(j) < hd;
                    kf[u][j] = ok ? k_s[elem(j)] : 0.f;
                    vf[u][j] = ok ? v_s[elem(j)] : 0.f;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kAttnUnroll; ++u) {
            const int t = tb + u * kAttnWarps;
            float dot = 0.f;
#pragma unroll
            for (int j = 0; j < PER; ++j) dot = fmaf(qr[j], kf[u][j], dot);
            dot = warp_sum(dot) * scale;
            if (t < t1) {  // warp-uniform
                const float m_new = fmaxf(m, dot);
                const float corr = expf(m - m_new);  // exp(-inf) = 0 on the first position
                const float pw = expf(dot - m_new);
                l = l * corr + pw;
#pragma unroll
                for (int j = 0; j < PER; ++j) acc[j] = acc[j] * corr + pw * vf[u][j];
                m = m_new;
            }
        }
    }
    if (lane == 0) {
        m_s[warp] = m;
        l_s[warp] = l;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j)
        if (elem(j) < hd) acc_s[warp][elem(j)] = acc[j];
    __syncthreads();
    // ---- merge the warps of this CTA ----
    float mm = -INFINITY;
#pragma unroll
    for (int wv = 0; wv < kAttnWarps; ++wv) mm = fmaxf(mm, m_s[wv]);
    float ll = 0.f;
#pragma unroll
    for (int wv = 0; wv < kAttnWarps; ++wv) ll += (m_s[wv] == -INFINITY) ? 0.f : l_s[wv] * expf(m_s[wv] - mm);
    if (n_split == 1) {
        for (int i = tid; i < hd; i += kAttnThreads) {
            float o = 0.f;
#pragma unroll
            for (int wv = 0; wv < kAttnWarps; ++wv)
                if (m_s[wv] != -INFINITY) o += acc_s[wv][i] * expf(m_s[wv] - mm);
            out[(long long)h * hd + i] = o / ll;
        }
        return;
    }
    // ---- partial of this split -> workspace; the last CTA of the head combines ----
    float* my = ws + ((long long)h * n_split + sp) * (hd + 2);
    for (int i = tid; i < hd; i += kAttnThreads) {
        float o = 0.f;
#pragma unroll
        for (int wv = 0; wv < kAttnWarps; ++wv)
            if (m_s[wv] != -INFINITY) o += acc_s[wv][i] * expf(m_s[wv] - mm);
        my[2 + i] = o;
    }
    if (tid == 0) {
        my[0] = mm;
        my[1] = ll;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = (atomicAdd(&tickets[h], 1) == n_split - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const float* hp = ws + (long long)h * n_split * (hd + 2);
    float gm = -INFINITY;
    for (int s2 = 0; s2 < n_split; ++s2) gm = fmaxf(gm, __ldcg(hp + (long long)s2 * (hd + 2)));
    float gl = 0.f;
    for (int s2 = 0; s2 < n_split; ++s2) {
        const float pm = __ldcg(hp + (long long)s2 * (hd + 2));
        if (pm != -INFINITY) gl += __ldcg(hp + (long long)s2 * (hd + 2) + 1) * expf(pm - gm);
    }
    for (int i = tid; i < hd; i += kAttnThreads) {
        float o = 0.f;
        for (int s2 = 0; s2 < n_split; ++s2) {
            const float pm = __ldcg(hp + (long long)s2 * (hd + 2));
            if (pm != -INFINITY) o += __ldcg(hp + (long long)s2 * (hd + 2) + 2 + i) * expf(pm - gm);
        }
        out[(long long)h * hd + i] = o / gl;
    }
    if (tid == 0) tickets[h] = 0;  // ready for the next launch (graph replay)
}

// ---- decode attention, second form: the KV chunk of a split is staged in shared memory with asynchronous
// 16-byte copies issued BEFORE griddepcontrol.wait ----
// The attention sits between two fused weight launches on the critical path of every layer, so what counts is
// its latency, not its bandwidth (16.8 MB of KV at 1024 positions of Llama-2-7B are 2.6 us of HBM time; the first
// kernel above takes 22.7 us there, 11 us at 128 positions: a chain of ~8 dependent global round trips).  Here:
//   * everything that does not depend on the previous kernel -- the position, the rotary row, and the split's
//     whole K/V chunk (positions < pos are static during a step) -- is requested before the wait for it;
//   * splits are 64 positions (16 at 1024, up to 32 per head), one position per warp and step, four steps
//     of dot products in flight per warp, so the serial online-softmax chain is 4 long per warp at 64 positions;
//   * the combine of a head's splits reads every partial in one batch of independent loads.
// hd = 64 or 128 (16-byte aligned caches); other head sizes keep attn_decode_kernel.
constexpr int kAt2Threads = 128;
constexpr int kAt2Warps = kAt2Threads / 32;
constexpr int kAt2Chunk = 64;          // positions per split (and per shared-memory chunk)
constexpr int kAt2MaxSplit = 32;

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int HD>
__global__ void __launch_bounds__(kAt2Threads) attn_decode2_kernel(const float* __restrict__ qkv, const long long* __restrict__ qkv_fix,
                                                                   const float* __restrict__ qkv_scale, __nv_bfloat16* __restrict__ k_cache,
                                                                   __nv_bfloat16* __restrict__ v_cache, const float* __restrict__ cos_t,
                                                                   const float* __restrict__ sin_t, const int32_t* __restrict__ pos_dev,
                                                                   int n_heads, int n_kv, int max_seq, float scale, int n_split,
                                                                   float* __restrict__ ws, int* __restrict__ tickets, float* __restrict__ out) {
    constexpr int EL = HD / 32;            // dims per lane (contiguous)
    constexpr int RC = HD / 8;             // 16-byte chunks per cached row
    constexpr int half = HD / 2;
    extern __shared__ __align__(16) unsigned char at2_smem[];
    __nv_bfloat16* kbuf = reinterpret_cast<__nv_bfloat16*>(at2_smem);                    // [kAt2Chunk][HD]
    __nv_bfloat16* vbuf = kbuf + kAt2Chunk * HD;
    __shared__ float q_s[HD], k_s[HD], v_s[HD];
    __shared__ float m_s[kAt2Warps], l_s[kAt2Warps];
    __shared__ float acc_s[kAt2Warps][HD];
    __shared__ float pm_s[kAt2MaxSplit], pl_s[kAt2MaxSplit];
    __shared__ int is_last;
    const int h = blockIdx.x / n_split, sp = blockIdx.x % n_split;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int group = n_heads / n_kv, kvh = h / group;
    // The position was written by the previous token's bookkeeping launch, which completed before this token's
    // first kernel started (the token boundary has plain launches): reading it ahead of the wait is safe.
    const int pos = *pos_dev;
    if (pos < 0 || pos >= max_seq) return;   // KV cache full: touch nothing (the host side raises StateError before it gets here)
    const int n_pos = pos + 1;
    n_split = min(n_split, max(1, (n_pos + kAt2Chunk - 1) / kAt2Chunk));
    if (sp >= n_split) return;
    const int per = (n_pos + n_split - 1) / n_split;
    const int t0 = sp * per, t1 = min(n_pos, t0 + per);
    const __nv_bfloat16* kbase = k_cache + (long long)kvh * max_seq * HD;
    const __nv_bfloat16* vbase = v_cache + (long long)kvh * max_seq * HD;
    auto prefetch = [&](int base) {
        const int n = min(kAt2Chunk, t1 - base);
        const uint32_t ks = smem_u32(kbuf), vs = smem_u32(vbuf);
        for (int idx = tid; idx < n * RC; idx += kAt2Threads) {
            const int r = idx / RC, c = idx % RC;
            const int t = base + r;
            if (t != pos) {   // the new position is not in the cache yet: it is used from k_s / v_s
                cp_async16(ks + (r * HD + c * 8) * 2, kbase + (long long)t * HD + c * 8);
                cp_async16(vs + (r * HD + c * 8) * 2, vbase + (long long)t * HD + c * 8);
            }
        }
        cp_async_commit();
    };
    prefetch(t0);
    float rc_ = 1.f, rs_ = 0.f;
    if (tid < half) {
        rc_ = __ldg(cos_t + (long long)pos * half + tid);
        rs_ = __ldg(sin_t + (long long)pos * half + tid);
    }
    pdl_wait();               // q | k | v of the new token come from the previous kernel
    pdl_launch_dependents();
    const long long oq = (long long)h * HD, ok = (long long)n_heads * HD + (long long)kvh * HD,
                    ov = (long long)(n_heads + n_kv) * HD + (long long)kvh * HD;
    const float fix_scale = (qkv_scale ? *qkv_scale : 1.0f) * (1.0f / (float)(1ll << AF_FIX_SHIFT));
    auto ld = [&](long long i) { return qkv_fix ? __ll2float_rn(__ldcg(qkv_fix + i)) * fix_scale : __ldcg(qkv + i); };
    if (tid < half) {   // RoPE (rotate-half); the cache stores bf16, and the new position uses the rounded values too
        const float q0 = ld(oq + tid), q1 = ld(oq + tid + half), k0 = ld(ok + tid), k1 = ld(ok + tid + half);
        q_s[tid] = q0 * rc_ - q1 * rs_;
        q_s[tid + half] = q1 * rc_ + q0 * rs_;
        k_s[tid] = __bfloat162float(__float2bfloat16_rn(k0 * rc_ - k1 * rs_));
        k_s[tid + half] = __bfloat162float(__float2bfloat16_rn(k1 * rc_ + k0 * rs_));
    }
    for (int i = tid; i < HD; i += kAt2Threads) v_s[i] = __bfloat162float(__float2bfloat16_rn(ld(ov + i)));
    __syncthreads();
    if (h % group == 0 && pos >= t0 && pos < t1) {  // one CTA per kv head appends to the cache
        __nv_bfloat16* kc = k_cache + ((long long)kvh * max_seq + pos) * HD;
        __nv_bfloat16* vc = v_cache + ((long long)kvh * max_seq + pos) * HD;
        for (int i = tid; i < HD; i += kAt2Threads) {
            kc[i] = __float2bfloat16_rn(k_s[i]);
            vc[i] = __float2bfloat16_rn(v_s[i]);
        }
    }
    float qr[EL], acc[EL];
#pragma unroll
    for (int j = 0; j < EL; ++j) {
        qr[j] = q_s[lane * EL + j] * scale;
        acc[j] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    for (int base = t0; base < t1; base += kAt2Chunk) {
        if (base > t0) {          // contexts beyond n_split * 64 positions: further chunks through the same buffer
            __syncthreads();
            prefetch(base);
        }
        cp_async_wait_all();
        __syncthreads();
        const int n = min(kAt2Chunk, t1 - base);
        constexpr int kFly = 4;   // positions per warp whose dot products are in flight together
        for (int r0 = warp; r0 < n; r0 += kAt2Warps * kFly) {
            float kf[kFly][EL], vf[kFly][EL], dot[kFly];
#pragma unroll
            for (int u = 0; u < kFly; ++u) {
                const int r = r0 + u * kAt2Warps;
                if (r < n && base + r != pos) {
                    load_bf16_vec<EL>(kbuf + r * HD + lane * EL, kf[u]);
                    load_bf16_vec<EL>(vbuf + r * HD + lane * EL, vf[u]);
                } else {
#pragma unroll
                    for (int j = 0; j < EL; ++j) {
                        kf[u][j] = r < n ? k_s[lane * EL + j] : 0.f;
                        vf[u][j] = r < n ? v_s[lane * EL + j] : 0.f;
                    }
                }
                float d = 0.f;
#pragma unroll
                for (int j = 0; j < EL; ++j) d = fmaf(qr[j], kf[u][j], d);
                dot[u] = d;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int u = 0; u < kFly; ++u) dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], o);
            float m_new = m;
#pragma unroll
            for (int u = 0; u < kFly; ++u)
                if (r0 + u * kAt2Warps < n) m_new = fmaxf(m_new, dot[u]);
            const float corr = expf(m - m_new);   // exp(-inf) = 0 on the first group
            l *= corr;
#pragma unroll
            for (int j = 0; j < EL; ++j) acc[j] *= corr;
#pragma unroll
            for (int u = 0; u < kFly; ++u)
                if (r0 + u * kAt2Warps < n) {     // warp-uniform
                    const float pw = expf(dot[u] - m_new);
                    l += pw;
#pragma unroll
                    for (int j = 0; j < EL; ++j) acc[j] = fmaf(pw, vf[u][j], acc[j]);
                }
            m = m_new;
        }
    }
    if (lane == 0) {
        m_s[warp] = m;
        l_s[warp] = l;
    }
#pragma unroll
    for (int j = 0; j < EL; ++j) acc_s[warp][lane * EL + j] = acc[j];
    __syncthreads();
    // ---- merge the warps of this CTA ----
    float mm = -INFINITY;
#pragma unroll
    for (int wv = 0; wv < kAt2Warps; ++wv) mm = fmaxf(mm, m_s[wv]);
    float ll = 0.f;
#pragma unroll
    for (int wv = 0; wv < kAt2Warps; ++wv) ll += (m_s[wv] == -INFINITY) ? 0.f : l_s[wv] * expf(m_s[wv] - mm);
    float o_part = 0.f;      // element tid of this split's un-normalised output (HD <= kAt2Threads)
    if (tid < HD) {
#pragma unroll
        for (int wv = 0; wv < kAt2Warps; ++wv)
            if (m_s[wv] != -INFINITY) o_part += acc_s[wv][tid] * expf(m_s[wv] - mm);
    }
    if (n_split == 1) {
        if (tid < HD) out[(long long)h * HD + tid] = o_part / ll;
        return;
    }
    // ---- partial of this split -> workspace; the last CTA of the head to arrive combines ----
    float* my = ws + ((long long)h * n_split + sp) * (HD + 2);
    if (tid < HD) my[2 + tid] = o_part;
    if (tid == 0) {
        my[0] = mm;
        my[1] = ll;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = (atomicAdd(&tickets[h], 1) == n_split - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    const float* hp = ws + (long long)h * n_split * (HD + 2);
    if (tid < n_split) {     // one batch of independent loads: every split's (max, sum) ...
        pm_s[tid] = __ldcg(hp + (long long)tid * (HD + 2));
        pl_s[tid] = __ldcg(hp + (long long)tid * (HD + 2) + 1);
    }
    float pv[kAt2MaxSplit];
    if (tid < HD) {          // ... and this thread's element of every partial
#pragma unroll
        for (int s2 = 0; s2 < kAt2MaxSplit; ++s2) pv[s2] = s2 < n_split ? __ldcg(hp + (long long)s2 * (HD + 2) + 2 + tid) : 0.f;
    }
    __syncthreads();
    float gm = -INFINITY;
    for (int s2 = 0; s2 < n_split; ++s2) gm = fmaxf(gm, pm_s[s2]);
    float gl = 0.f, o = 0.f;
#pragma unroll
    for (int s2 = 0; s2 < kAt2MaxSplit; ++s2)
        if (s2 < n_split && pm_s[s2] != -INFINITY) {
            const float e = expf(pm_s[s2] - gm);
            gl += pl_s[s2] * e;
            o += pv[s2] * e;
        }
    if (tid < HD) out[(long long)h * HD + tid] = o / gl;
    if (tid == 0) tickets[h] = 0;  // ready for the next launch (graph replay)
}

// out[i] = (res ? res[i] : 0) + fixed-point accumulator i (the residual stream after the last fused
// switch + GEMV launch, as a plain f32 vector for the lm_head GEMV).
__global__ void accum_to_f32_kernel(const long long* __restrict__ acc, const float* __restrict__ res, float* __restrict__ out, int n) {
    pdl_wait();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = (res ? res[i] : 0.f) + __ll2float_rn(acc[i]) * (1.0f / (float)(1ll << AF_FIX_SHIFT));
}

// argmax with the winning value (vocab-parallel lm_head: ranks exchange (value, index)).
__global__ void __launch_bounds__(1024) argmax_val_kernel(const float* __restrict__ v, int n, int index_offset,
                                                          int32_t* __restrict__ out_idx, float* __restrict__ out_val) {
    __shared__ float sv[32];
    __shared__ int si[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float best = -INFINITY;
    int best_i = 0x7fffffff;
    // 8 loads in flight per thread (one load per iteration is a chain of L2 round trips: 32 of them at 32000 entries);
    // a thread's indices ascend, so the strict > keeps the lowest index among equal values
    constexpr int kFly = 8;
    for (int base = tid; base < n; base += kFly * blockDim.x) {
        float x[kFly];
#pragma unroll
        for (int u = 0; u < kFly; ++u) {
            const int i = base + u * blockDim.x;
            x[u] = i < n ? v[i] : -INFINITY;
        }
#pragma unroll
        for (int u = 0; u < kFly; ++u) {
            const int i = base + u * blockDim.x;
            if (i < n && (best_i == 0x7fffffff || x[u] > best)) { best = x[u]; best_i = i; }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (oi != 0x7fffffff && (best_i == 0x7fffffff || ov > best || (ov == best && oi < best_i))) { best = ov; best_i = oi; }
    }
    if (lane == 0) { sv[warp] = best; si[warp] = best_i; }
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        best = lane < nw ? sv[lane] : -INFINITY;
        best_i = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
            if (oi != 0x7fffffff && (best_i == 0x7fffffff || ov > best || (ov == best && oi < best_i))) { best = ov; best_i = oi; }
        }
        if (lane == 0) {
            *out_idx = (best_i == 0x7fffffff ? 0 : best_i) + index_offset;
            if (out_val) *out_val = best;
        }
    }
}

// End-of-step bookkeeping, one tiny launch so a whole decode step is a static CUDA graph:
//   prev decision <- cur decision; position += 1; steps += 1;
//   consumed token <- forced[steps] when a teacher-forced stream is given, else the argmax.
__global__ void step_advance_kernel(af_decision* __restrict__ prev, const af_decision* __restrict__ cur,
                                    int32_t* __restrict__ pos_dev, int32_t* __restrict__ step_dev,
                                    int32_t* __restrict__ token_dev, const int32_t* __restrict__ next_dev,
                                    const int32_t* __restrict__ forced, int n_forced, int32_t* __restrict__ history,
                                    int n_history) {
    const int tid = threadIdx.x;
    if (prev && cur && tid < (int)(sizeof(af_decision) / 4))
        reinterpret_cast<int32_t*>(prev)[tid] = reinterpret_cast<const int32_t*>(cur)[tid];
    if (tid == 0) {
        const int step = *step_dev;
        if (history && step < n_history) history[step] = *next_dev;
        if (pos_dev) *pos_dev += 1;
        *step_dev = step + 1;
        if (forced && n_forced > 0) *token_dev = forced[(step + 1) % n_forced];
        else *token_dev = *next_dev;
    }
}

}  // namespace af
