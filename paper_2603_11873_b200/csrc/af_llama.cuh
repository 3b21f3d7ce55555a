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

constexpr int kGemvFThreads = 256;
constexpr int kGemvFRows = 2;  // rows per warp per pass

__device__ __forceinline__ void unpack8(const uint4 v, float (&f)[8]) {
    f[0] = bf16lo_to_f32(v.x); f[1] = bf16hi_to_f32(v.x); f[2] = bf16lo_to_f32(v.y); f[3] = bf16hi_to_f32(v.y);
    f[4] = bf16lo_to_f32(v.z); f[5] = bf16hi_to_f32(v.z); f[6] = bf16lo_to_f32(v.w); f[7] = bf16hi_to_f32(v.w);
}

// Streaming 16-byte load that does not pollute L1 (W is read exactly once per token).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// y = W xs, W rows x cols bf16 row-major (cols % 8 == 0, 16-byte aligned rows), x f32.
// Each CTA stages xs once (prologue applied) and grid-strides over row groups; a warp owns
// kGemvFRows rows per pass, lanes stride the row in 16-byte chunks, 4 chunks per row in
// flight (8 independent 16-byte loads per thread), f32 FMA, shuffle tree, epilogue by lane 0.
__global__ void __launch_bounds__(kGemvFThreads) gemv_fused_kernel(const __nv_bfloat16* __restrict__ w, int rows, int cols,
                                                                    long long ld, const float* __restrict__ x,
                                                                    float* __restrict__ out, int prologue,
                                                                    const float* __restrict__ norm_w, float eps, int epilogue,
                                                                    const float* __restrict__ res) {
    extern __shared__ __align__(16) float xs[];
    __shared__ float red[kGemvFThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kGemvFThreads / 32;
    if (prologue == kPrologueRmsNorm) {
        float ss = 0.f;
        for (int c = tid; c < cols; c += kGemvFThreads) {
            const float v = x[c];
            xs[c] = v;
            ss = fmaf(v, v, ss);
        }
        ss = warp_sum(ss);
        if (lane == 0) red[warp] = ss;
        __syncthreads();
        float tot = 0.f;
#pragma unroll
        for (int i = 0; i < nwarps; ++i) tot += red[i];
        const float inv = rsqrtf(tot / (float)cols + eps);
        for (int c = tid; c < cols; c += kGemvFThreads) xs[c] = xs[c] * inv * norm_w[c];
    } else if (prologue == kPrologueSiluMul) {
        for (int c = tid; c < cols; c += kGemvFThreads) {
            const float g = x[c], u = x[cols + c];
            xs[c] = g / (1.0f + expf(-g)) * u;
        }
    } else {
        for (int c = tid; c < cols; c += kGemvFThreads) xs[c] = x[c];
    }
    __syncthreads();
    const int rows_per_cta = nwarps * kGemvFRows;
    for (int r0 = blockIdx.x * rows_per_cta + warp * kGemvFRows; r0 < rows; r0 += gridDim.x * rows_per_cta) {
        float acc[kGemvFRows] = {};
        const __nv_bfloat16* wr[kGemvFRows];
#pragma unroll
        for (int i = 0; i < kGemvFRows; ++i) wr[i] = w + (long long)min(r0 + i, rows - 1) * ld;
        int c = lane * 8;
        for (; c + 3 * 256 < cols; c += 4 * 256) {
            uint4 v[kGemvFRows][4];
#pragma unroll
            for (int i = 0; i < kGemvFRows; ++i)
#pragma unroll
                for (int u = 0; u < 4; ++u) v[i][u] = ldg_stream(wr[i] + c + u * 256);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float4 xa = *reinterpret_cast<const float4*>(xs + c + u * 256);
                const float4 xb = *reinterpret_cast<const float4*>(xs + c + u * 256 + 4);
                const float xf[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
                for (int i = 0; i < kGemvFRows; ++i) {
                    float wf[8];
                    unpack8(v[i][u], wf);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i] = fmaf(wf[j], xf[j], acc[i]);
                }
            }
        }
        for (; c < cols; c += 256) {
            const float4 xa = *reinterpret_cast<const float4*>(xs + c);
            const float4 xb = *reinterpret_cast<const float4*>(xs + c + 4);
            const float xf[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
            for (int i = 0; i < kGemvFRows; ++i) {
                float wf[8];
                unpack8(ldg_stream(wr[i] + c), wf);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i] = fmaf(wf[j], xf[j], acc[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < kGemvFRows; ++i) {
            const float y = warp_sum(acc[i]);
            if (lane == 0 && r0 + i < rows) {
                float o = y;
                if (epilogue == AF_EPI_GELU_RESIDUAL)
                    o = res[r0 + i] + 0.5f * y * (1.0f + erff(y * 0.70710678118654752440f));
                else if (epilogue == AF_EPI_RESIDUAL)
                    o = res[r0 + i] + y;
                out[r0 + i] = o;
            }
        }
    }
}

// Single-query GQA attention for one new token, fused with RoPE and the KV-cache append.
//   qkv     : f32 [n_heads*hd | n_kv*hd | n_kv*hd]  (output of the fused q/k/v GEMV)
//   k_cache : bf16 [n_kv][max_seq][hd], v_cache likewise; position *pos_dev is written here
//   cos/sin : f32 [max_seq][hd/2] rotary tables (rotate-half convention)
//   out     : f32 [n_heads*hd]
// One CTA per query head.  The head's own (rotated) k and v of the new position are used from
// shared memory, so heads of one group never read what a sibling CTA is still writing.
constexpr int kAttnThreads = 128;
constexpr int kAttnMaxHd = 256;

__global__ void __launch_bounds__(kAttnThreads) attn_decode_kernel(const float* __restrict__ qkv,
                                                                   __nv_bfloat16* __restrict__ k_cache,
                                                                   __nv_bfloat16* __restrict__ v_cache,
                                                                   const float* __restrict__ cos_t,
                                                                   const float* __restrict__ sin_t,
                                                                   const int32_t* __restrict__ pos_dev, int n_heads,
                                                                   int n_kv, int hd, int max_seq, float scale,
                                                                   float* __restrict__ out) {
    __shared__ float q_s[kAttnMaxHd], k_s[kAttnMaxHd], v_s[kAttnMaxHd];
    __shared__ float m_s[kAttnThreads / 32], l_s[kAttnThreads / 32];
    __shared__ float acc_s[kAttnThreads / 32][kAttnMaxHd];
    const int h = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = kAttnThreads / 32;
    const int group = n_heads / n_kv, kvh = h / group;
    const int pos = *pos_dev;
    const int half = hd >> 1;
    const float* q = qkv + (long long)h * hd;
    const float* kn = qkv + (long long)n_heads * hd + (long long)kvh * hd;
    const float* vn = qkv + (long long)(n_heads + n_kv) * hd + (long long)kvh * hd;
    // RoPE (rotate-half): x'[i] = x[i] c - x[i+half] s ; x'[i+half] = x[i+half] c + x[i] s
    for (int i = tid; i < half; i += kAttnThreads) {
        const float c = cos_t[(long long)pos * half + i], s = sin_t[(long long)pos * half + i];
        const float q0 = q[i], q1 = q[i + half];
        q_s[i] = q0 * c - q1 * s;
        q_s[i + half] = q1 * c + q0 * s;
        const float k0 = kn[i], k1 = kn[i + half];
        // the cache stores bf16: use the rounded values for the new position too, so that a
        // later token sees exactly what this one saw
        k_s[i] = __bfloat162float(__float2bfloat16_rn(k0 * c - k1 * s));
        k_s[i + half] = __bfloat162float(__float2bfloat16_rn(k1 * c + k0 * s));
    }
    for (int i = tid; i < hd; i += kAttnThreads) v_s[i] = __bfloat162float(__float2bfloat16_rn(vn[i]));
    __syncthreads();
    if (h % group == 0) {  // one head per group appends to the cache
        __nv_bfloat16* kc = k_cache + ((long long)kvh * max_seq + pos) * hd;
        __nv_bfloat16* vc = v_cache + ((long long)kvh * max_seq + pos) * hd;
        for (int i = tid; i < hd; i += kAttnThreads) {
            kc[i] = __float2bfloat16_rn(k_s[i]);
            vc[i] = __float2bfloat16_rn(v_s[i]);
        }
    }
    // online softmax over positions 0..pos; warp w takes positions w, w+nwarps, ...
    // lane owns elements lane, lane+32, ... of the head dimension
    constexpr int kPer = kAttnMaxHd / 32;
    float acc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[j] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int t = warp; t <= pos; t += nwarps) {
        float dot = 0.f;
        float vv[kPer];
        if (t == pos) {
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const int i = lane + 32 * j;
                if (i < hd) {
                    dot = fmaf(q_s[i], k_s[i], dot);
                    vv[j] = v_s[i];
                }
            }
        } else {
            const __nv_bfloat16* kc = k_cache + ((long long)kvh * max_seq + t) * hd;
            const __nv_bfloat16* vc = v_cache + ((long long)kvh * max_seq + t) * hd;
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const int i = lane + 32 * j;
                if (i < hd) {
                    dot = fmaf(q_s[i], __bfloat162float(kc[i]), dot);
                    vv[j] = __bfloat162float(vc[i]);
                }
            }
        }
        dot = warp_sum(dot) * scale;
        const float m_new = fmaxf(m, dot);
        const float corr = expf(m - m_new);  // exp(-inf) = 0 on the first position
        const float p = expf(dot - m_new);
        l = l * corr + p;
#pragma unroll
        for (int j = 0; j < kPer; ++j)
            if (lane + 32 * j < hd) acc[j] = acc[j] * corr + p * vv[j];
        m = m_new;
    }
    if (lane == 0) {
        m_s[warp] = m;
        l_s[warp] = l;
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j)
        if (lane + 32 * j < hd) acc_s[warp][lane + 32 * j] = acc[j];
    __syncthreads();
    float mm = -INFINITY;
    for (int wv = 0; wv < nwarps; ++wv) mm = fmaxf(mm, m_s[wv]);
    float ll = 0.f;
    for (int wv = 0; wv < nwarps; ++wv) ll += (m_s[wv] == -INFINITY) ? 0.f : l_s[wv] * expf(m_s[wv] - mm);
    for (int i = tid; i < hd; i += kAttnThreads) {
        float o = 0.f;
        for (int wv = 0; wv < nwarps; ++wv)
            if (m_s[wv] != -INFINITY) o += acc_s[wv][i] * expf(m_s[wv] - mm);
        out[(long long)h * hd + i] = o / ll;
    }
}

// argmax with the winning value (vocab-parallel lm_head: ranks exchange (value, index)).
__global__ void __launch_bounds__(1024) argmax_val_kernel(const float* __restrict__ v, int n, int index_offset,
                                                          int32_t* __restrict__ out_idx, float* __restrict__ out_val) {
    __shared__ float sv[32];
    __shared__ int si[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float best = -INFINITY;
    int best_i = 0x7fffffff;
    for (int i = tid; i < n; i += blockDim.x) {
        const float x = v[i];
        if (best_i == 0x7fffffff || x > best) { best = x; best_i = i; }
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
