// af_decode.cuh -- pre-gating router and the bs=1 decode kernels.
//
//   pregate_kernel  routing.py:49-78 `route`: N dot products (GEMV), stable top-k, softmax over
//                   the selected logits, fused with the embedding-row gather of model.py:248-258.
//   gemv_kernel     linalg.py:246-259 `gemm` as y = W x with the GELU+residual of
//                   model.py:298-305 fused into the epilogue.
//   gemv_t_kernel   model.py:261-263 `_unembed`: y = W^T x.
//   argmax_kernel   model.py:396 `np.argmax` (lowest index on ties).
#pragma once

#include "af_common.cuh"

namespace af {

// ------------------------------------------------------------------ router ----
// One CTA.  Warp w scores experts w, w+nwarps, ...; each lane owns 8-element chunks
// lane, lane+32, ... of the row.  Products of bf16 values are exact in f64 and the f64 sum is
// order independent to ~1e-16 relative, so the logit, rounded ONCE to f32, does not depend on
// the reduction tree -- that is what makes the expert ids reproducible bit for bit against the
// CPU oracle.  Top-k: descending logit, ascending index on ties
// (routing.py:64-65).  Softmax over the k selected logits only, max-shifted (routing.py:66-68),
// evaluated in f64 and rounded once to f32.

constexpr int kRouterThreads = 512;
constexpr int kRouterMaxExperts = 256;

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&f)[8]);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    f[0] = bf16lo_to_f32(v.x); f[1] = bf16hi_to_f32(v.x); f[2] = bf16lo_to_f32(v.y); f[3] = bf16hi_to_f32(v.y);
    f[4] = bf16lo_to_f32(v.z); f[5] = bf16hi_to_f32(v.z); f[6] = bf16lo_to_f32(v.w); f[7] = bf16hi_to_f32(v.w);
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&f)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// Order of `np.argsort(-logits, kind="stable")` (routing.py:64-65): larger logit first, equal logits (+0 == -0)
// by index, NaN after every number (numpy sorts NaN last), NaN against NaN by index.
__device__ __forceinline__ bool router_better(float v, int id, float best, int best_id) {
    if (id == 0x7fffffff) return false;
    if (best_id == 0x7fffffff) return true;
    const bool vn = v != v, bn = best != best;
    if (vn != bn) return bn;
    if (vn) return id < best_id;
    return v > best || (v == best && id < best_id);
}

template <typename WT, typename XT>
__global__ void __launch_bounds__(kRouterThreads) pregate_kernel(const WT* __restrict__ wg, int n_experts, int d,
                                                                 const XT* __restrict__ x_base,
                                                                 const int32_t* __restrict__ token_dev, int k,
                                                                 af_decision* __restrict__ out,
                                                                 float* __restrict__ logits_out) {
    __shared__ float logits[kRouterMaxExperts];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const XT* x = x_base + (token_dev ? (long long)(*token_dev) * d : 0ll);
    const bool vec = (d % 8 == 0) && ((reinterpret_cast<uintptr_t>(wg) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && sizeof(XT) * 8 % 16 == 0;
    for (int e = warp; e < n_experts; e += nwarps) {
        const WT* row = wg + (long long)e * d;
        double acc = 0.0;
        if (vec) {
            for (int c = lane * 8; c < d; c += 256) {
                float wf[8], xf[8];
                load8<WT>(row + c, wf);
                load8<XT>(x + c, xf);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc = fma((double)wf[j], (double)xf[j], acc);
            }
        } else {
            for (int c = lane; c < d; c += 32) acc = fma((double)load_as_f32<WT>(row + c), (double)load_as_f32<XT>(x + c), acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) logits[e] = (float)acc;  // single rounding
    }
    __syncthreads();
    if (logits_out)
        for (int e = tid; e < n_experts; e += blockDim.x) logits_out[e] = logits[e];
    if (warp != 0) return;
    // ---- top-k by k rounds of (max value, min index) over the not-yet-taken experts ----
    unsigned taken_mask[kRouterMaxExperts / 32] = {};  // lane-local view: bit j <-> expert lane + 32*j
    float sel_logit = 0.f;  // lane j < k keeps the j-th selected logit
    int sel_id = 0;
    for (int j = 0; j < k; ++j) {
        float best = -INFINITY;
        int best_id = 0x7fffffff;
        for (int s = 0, e = lane; e < n_experts; e += 32, ++s) {
            if (taken_mask[s >> 5] & (1u << (s & 31))) continue;
            const float v = logits[e];
            if (router_better(v, e, best, best_id)) { best = v; best_id = e; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, best_id, o);
            if (router_better(ov, oi, best, best_id)) {
                best = ov;
                best_id = oi;
            }
        }
        if ((best_id & 31) == lane) {
            const int s = best_id >> 5;
            taken_mask[s >> 5] |= 1u << (s & 31);
        }
        if (lane == j) { sel_logit = best; sel_id = best_id; }
    }
    // ---- softmax over the selected logits (routing.py:66-68), max-shifted.  exp, the
    //      left-to-right sum and the division run in f64 and round ONCE to f32: the result is
    //      the correctly rounded f32 softmax, within 1 f32 ulp of any f32 evaluation (numpy's,
    //      glibc's, CUDA's differ among themselves by that much) and identical on CPU and GPU. ----
    const float mx = __shfl_sync(0xffffffffu, sel_logit, 0);  // first selected is the maximum
    const double ex = lane < k ? exp((double)sel_logit - (double)mx) : 0.0;
    double total = 0.0;
    for (int j = 0; j < k; ++j) total += __shfl_sync(0xffffffffu, ex, j);
    const float wgt = (float)(ex / total);
    if (lane < k) {
        out->ids[lane] = sel_id;
        out->weights[lane] = wgt;
    } else if (lane < AF_MAX_K) {
        out->ids[lane] = -1;
        out->weights[lane] = 0.f;
    }
    if (lane == 0) out->k = k;
}

// -------------------------------------------------------------------- GEMV ----
// y = W x, W: rows x cols bf16/f32 row-major (pitch ld), x: f32[cols].  HBM-bound streaming
// read of W.  x is staged once per CTA in shared memory as f32; each warp owns kRowsPerWarp
// rows at a time and its lanes stride the row in 16-byte chunks (coalesced 512 B per warp
// request), f32 FMA accumulation, warp-shuffle tree, epilogue by lane 0.

constexpr int kGemvThreads = 256;
constexpr int kRowsPerWarp = 2;

template <typename WT>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(const WT* __restrict__ w, int rows, int cols, long long ld,
                                                            const float* __restrict__ x, float* __restrict__ out,
                                                            int epilogue, const float* __restrict__ res) {
    extern __shared__ __align__(16) float xs[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int c = tid; c < cols; c += blockDim.x) xs[c] = x[c];
    __syncthreads();
    const bool vec = (cols % 8 == 0) && (ld % 8 == 0) && ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
    const int rows_per_cta = nwarps * kRowsPerWarp;
    for (int r0 = blockIdx.x * rows_per_cta + warp * kRowsPerWarp; r0 < rows; r0 += gridDim.x * rows_per_cta) {
        float acc[kRowsPerWarp];
#pragma unroll
        for (int i = 0; i < kRowsPerWarp; ++i) acc[i] = 0.f;
        if (vec) {
            for (int c = lane * 8; c < cols; c += 256) {
                const float4 xa = *reinterpret_cast<const float4*>(xs + c);
                const float4 xb = *reinterpret_cast<const float4*>(xs + c + 4);
                const float xf[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
                for (int i = 0; i < kRowsPerWarp; ++i) {
                    if (r0 + i < rows) {
                        float wf[8];
                        load8<WT>(w + (long long)(r0 + i) * ld + c, wf);
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[i] = fmaf(wf[j], xf[j], acc[i]);
                    }
                }
            }
        } else {
            for (int c = lane; c < cols; c += 32)
#pragma unroll
                for (int i = 0; i < kRowsPerWarp; ++i)
                    if (r0 + i < rows) acc[i] = fmaf(load_as_f32<WT>(w + (long long)(r0 + i) * ld + c), xs[c], acc[i]);
        }
#pragma unroll
        for (int i = 0; i < kRowsPerWarp; ++i) {
            const float y = warp_sum(acc[i]);
            if (lane == 0 && r0 + i < rows) {
                float o = y;
                if (epilogue == AF_EPI_GELU_RESIDUAL)
                    o = res[r0 + i] + 0.5f * y * (1.0f + erff(y * 0.70710678118654752440f));  // model.py:245,305
                else if (epilogue == AF_EPI_RESIDUAL)
                    o = res[r0 + i] + y;
                out[r0 + i] = o;
            }
        }
    }
}

// y = W^T x: W rows x cols row-major, x f32[rows], y f32[cols].  Thread t of a CTA owns 8
// consecutive columns; the CTA's warps split the rows and combine through shared memory.
constexpr int kGemvTThreads = 256;
constexpr int kGemvTCols = 256;  // columns per CTA: 32 lanes x 8

template <typename WT>
__global__ void __launch_bounds__(kGemvTThreads) gemv_t_kernel(const WT* __restrict__ w, int rows, int cols, long long ld,
                                                               const float* __restrict__ x, float* __restrict__ out) {
    __shared__ float part[kGemvTThreads / 32][kGemvTCols];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int c0 = blockIdx.x * kGemvTCols + lane * 8;
    const bool vec = (cols % 8 == 0) && (ld % 8 == 0) && ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = warp; r < rows; r += nwarps) {
        const float xv = __ldg(x + r);
        if (vec) {
            if (c0 < cols) {
                float wf[8];
                load8<WT>(w + (long long)r * ld + c0, wf);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = fmaf(wf[j], xv, acc[j]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c0 + j < cols) acc[j] = fmaf(load_as_f32<WT>(w + (long long)r * ld + c0 + j), xv, acc[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) part[warp][lane * 8 + j] = acc[j];
    __syncthreads();
    for (int c = tid; c < kGemvTCols; c += blockDim.x) {
        float s = 0.f;
        for (int wv = 0; wv < nwarps; ++wv) s += part[wv][c];
        const int col = blockIdx.x * kGemvTCols + c;
        if (col < cols) out[col] = s;
    }
}

// ------------------------------------------------------------------ argmax ----
__global__ void __launch_bounds__(1024) argmax_kernel(const float* __restrict__ v, int n, int32_t* __restrict__ out) {
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
        if (lane == 0) *out = best_i == 0x7fffffff ? 0 : best_i;
    }
}

// model.py:248-258 `_embed_token`: row gather, widened to f32.
template <typename T>
__global__ void embed_kernel(const T* __restrict__ table, int d, const int32_t* __restrict__ token_dev,
                             float* __restrict__ out) {
    const T* row = table + (long long)(*token_dev) * d;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) out[i] = load_as_f32<T>(row + i);
}

// max |live - pristine| over a table (model.py:231-236), result via atomicMax on the
// non-negative float's bit pattern.
template <typename WT>
__global__ void max_dev_kernel(const WT* __restrict__ a, const WT* __restrict__ b, int rows, int cols, long long ld,
                               unsigned* __restrict__ out_bits) {
    float worst = 0.f;
    const long long n = (long long)rows * cols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cols, c = i % cols;
        const float dlt = fabsf(load_as_f32<WT>(a + r * ld + c) - load_as_f32<WT>(b + r * ld + c));
        worst = fmaxf(worst, dlt);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) worst = fmaxf(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, __float_as_uint(worst));
}

}  // namespace af
