// af_gemv_chain.cuh -- the merged-path forward (model.py:367-368 on the Llama block) between two
// attentions as ONE persistent launch: o -> gate|up -> down -> next layer's q|k|v (or lm_head).
//
// The projections depend on each other, but their WEIGHTS do not depend on anything: a producer
// warp streams every phase's rows through one shared-memory ring with 1-D bulk copies and never
// stops at a phase boundary, so HBM stays busy while the consumers wait for the previous phase's
// outputs (a device counter every CTA bumps), rebuild the input vector (RMSNorm / SiLU*up) and
// catch up -- they dot a 32 KB stage 3x faster than HBM delivers one.  Per-launch start-up and
// drain, which cost the one-GEMV-per-launch chain a third of its time at bs = 1, are paid once
// per layer instead of four times.
//
// Work split: phase rows are divided evenly over the CTAs; a CTA takes its rows in groups of 8, one
// kGcCH-column chunk of the group per ring stage.  Warp w sums columns [256 w, 256 w + 256) of every
// chunk for all 8 rows; lanes are combined by shuffles, warps in a fixed order through shared
// memory (deterministic, no atomics).
#pragma once

#include "af_llama.cuh"

namespace af {

constexpr int kGcWarps = 8;                        // rows per group = 256-column slices per 2048 columns
#ifndef AF_GC_HALVES
#define AF_GC_HALVES 2
#endif
constexpr int kGcHalves = AF_GC_HALVES;            // consumer warps per column slice, each taking 8 / kGcHalves rows
constexpr int kGcCons = kGcWarps * kGcHalves;      // consumer warps
#ifndef AF_GC_PROD
#define AF_GC_PROD 2
#endif
#ifndef AF_GC_CH
#define AF_GC_CH 2048
#endif
constexpr int kGcProd = AF_GC_PROD;                // producer threads (one per warp)
constexpr int kGcCH = AF_GC_CH;                    // columns per bulk copy (4 KB)
constexpr int kGcStage = kGcWarps * kGcCH * 2;     // 32 KB
constexpr int kGcMaxStages = 12;
constexpr int kGcMaxPhases = 4;
constexpr int kGcThreads = (kGcCons + kGcProd) * 32;
static_assert(kGcCH % 2048 == 0, "a chunk is a whole number of 8 x 256-column warp slices");

struct GcPhase {
    const __nv_bfloat16* w;
    int rows, cols;
    long long ld;
    const float* x;        // input vector (2 * cols entries for SILU_MUL)
    float* out;
    const float* res;      // epilogue residual (AF_EPI_RESIDUAL)
    const float* norm_w;
    float eps;
    int prologue, epilogue;
};

struct GcParams {
    GcPhase ph[kGcMaxPhases];
    int n_phases;
    int* phase_done;       // [n_phases - 1], zeroed by the caller
    int n_stages;
    int pdl;
    int* err_flag;
};

__global__ void __launch_bounds__(kGcThreads, 1) gemv_chain_kernel(const __grid_constant__ GcParams gp) {
    extern __shared__ __align__(128) unsigned char gc_smem[];
    __shared__ uint64_t full[kGcMaxStages], empty[kGcMaxStages];
    __shared__ float redn[kGcCons];
    __shared__ float gpart[2 * kGcWarps * kGcWarps];   // per-warp partial sums of a row group, double buffered
    const int n_stages = gp.n_stages;
    float* xs = reinterpret_cast<float*>(gc_smem + (size_t)n_stages * kGcStage);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = (int)gridDim.x;
    if (tid == 0) {
        for (int s = 0; s < n_stages; ++s) {
            mbar_init(&full[s], kGcProd);
            mbar_init(&empty[s], kGcCons);
        }
        fence_mbar_init();
    }
    __syncthreads();

    auto row_begin = [&](const GcPhase& f, int c) { return (int)((long long)f.rows * c / G); };

    if (warp >= kGcCons) {
        // ===================== producers: stream W of every phase, never blocked by a phase boundary ==========
        if (lane == 0) {
            const int who = warp - kGcCons;
            const uint32_t base = smem_u32(gc_smem);
            int it = 0;
            for (int p = 0; p < gp.n_phases; ++p) {
                const GcPhase& f = gp.ph[p];
                const int r_begin = row_begin(f, blockIdx.x), r_end = row_begin(f, blockIdx.x + 1);
                const int n_ch = (f.cols + kGcCH - 1) / kGcCH;
                for (int row0 = r_begin; row0 < r_end; row0 += kGcWarps) {
                    const int nrow = min(kGcWarps, r_end - row0);
                    for (int ch = 0; ch < n_ch; ++ch, ++it) {
                        const int stage = it % n_stages;
                        const uint32_t par = (it / n_stages) & 1;
                        const int c0 = ch * kGcCH;
                        const uint32_t bytes = (uint32_t)min(kGcCH, f.cols - c0) * 2;
                        int mine = 0;
                        for (int r = who; r < nrow; r += kGcProd) ++mine;
                        mbar_wait(&empty[stage], par ^ 1);
                        mbar_expect_tx(&full[stage], bytes * mine);
                        for (int r = who; r < nrow; r += kGcProd)
                            gv_bulk_load(base + stage * kGcStage + r * (kGcCH * 2), f.w + (long long)(row0 + r) * f.ld + c0, bytes,
                                         &full[stage]);
                    }
                }
            }
        }
        return;
    }

    // ===================== consumers =====================
    constexpr int kC = kGcCons * 32;
    constexpr int kRowsPer = kGcWarps / kGcHalves;   // rows of a group this warp sums
    const int slice = warp % kGcWarps, rbase = (warp / kGcWarps) * kRowsPer;
    if (gp.pdl) {
        pdl_wait();  // the first phase's input comes from the previous kernel
        if (tid == 0) pdl_launch_dependents();
    }
    int it = 0;
    for (int p = 0; p < gp.n_phases; ++p) {
        const GcPhase& f = gp.ph[p];
        if (p > 0) {
            // every CTA has written its rows of phase p - 1
            if (tid == 0) {
                const long long t0 = clock64();
                int seen;
                unsigned spins = 0;
                do {
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(gp.phase_done + p - 1) : "memory");
                    if (seen >= G) break;
                    // ~2 s: never hang the device on a lost CTA.  The first CTA to give up raises AF_ECUDA in the
                    // caller's error word; every other CTA sees the word and stops waiting at once, so the launch
                    // ends (with unusable outputs) and the host raises at its next status check.
                    if ((++spins & 1023u) == 0 && gp.err_flag && *reinterpret_cast<volatile int*>(gp.err_flag) == AF_ECUDA) break;
                    if (clock64() - t0 > (1ll << 32)) {
                        if (gp.err_flag) atomicExch(gp.err_flag, AF_ECUDA);
                        break;
                    }
                } while (true);
            }
            named_bar_sync(1, kC);
        }
        // ---- input vector of the phase -> shared memory (through L2: other CTAs wrote it in this launch) ----
        const int cols = f.cols;
        if (f.prologue == AF_PRO_RMSNORM) {
            float ss = 0.f;
            for (int c = tid * 4; c < cols; c += kC * 4) {
                const float4 v = __ldcg(reinterpret_cast<const float4*>(f.x + c));
                *reinterpret_cast<float4*>(xs + c) = v;
                ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
            }
            ss = warp_sum(ss);
            if (lane == 0) redn[warp] = ss;
            named_bar_sync(1, kC);
            float tot = 0.f;
#pragma unroll
            for (int i = 0; i < kGcCons; ++i) tot += redn[i];
            const float inv = rsqrtf(tot / (float)cols + f.eps);
            for (int c = tid * 4; c < cols; c += kC * 4) {
                float4 v = *reinterpret_cast<float4*>(xs + c);
                const float4 nw = *reinterpret_cast<const float4*>(f.norm_w + c);
                v.x *= inv * nw.x; v.y *= inv * nw.y; v.z *= inv * nw.z; v.w *= inv * nw.w;
                *reinterpret_cast<float4*>(xs + c) = v;
            }
        } else if (f.prologue == AF_PRO_SILU_MUL) {
            // four steps of loads in flight per thread: the boundary is one L2 round trip, not one per step
            for (int base = tid * 4; base < cols; base += 4 * kC * 4) {
                float4 g[4], u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int c = base + k * kC * 4;
                    if (c < cols) {
                        g[k] = __ldcg(reinterpret_cast<const float4*>(f.x + c));
                        u[k] = __ldcg(reinterpret_cast<const float4*>(f.x + cols + c));
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int c = base + k * kC * 4;
                    if (c < cols) {
                        float4 v;
                        v.x = g[k].x / (1.0f + expf(-g[k].x)) * u[k].x;
                        v.y = g[k].y / (1.0f + expf(-g[k].y)) * u[k].y;
                        v.z = g[k].z / (1.0f + expf(-g[k].z)) * u[k].z;
                        v.w = g[k].w / (1.0f + expf(-g[k].w)) * u[k].w;
                        *reinterpret_cast<float4*>(xs + c) = v;
                    }
                }
            }
        } else {
            for (int c = tid * 4; c < cols; c += kC * 4)
                *reinterpret_cast<float4*>(xs + c) = __ldcg(reinterpret_cast<const float4*>(f.x + c));
        }
        named_bar_sync(1, kC);

        // ---- this CTA's rows in groups of 8; a stage holds one kGcCH-column chunk of the 8 rows.  Warp w
        //      owns columns [256 w, 256 w + 256) of the chunk for ALL 8 rows: its 8 x values per lane are
        //      loaded once per stage and reused by every row (x is read from shared memory 8x less often
        //      than with one row per warp, which made the consumers shared-memory-bound at HBM speed) ----
        const int r_begin = row_begin(f, blockIdx.x), r_end = row_begin(f, blockIdx.x + 1);
        const int n_ch = (cols + kGcCH - 1) / kGcCH;
        int grp = 0;
        for (int row0 = r_begin; row0 < r_end; row0 += kGcWarps, ++grp) {
            float acc[kRowsPer];
#pragma unroll
            for (int r = 0; r < kRowsPer; ++r) acc[r] = 0.f;
            for (int ch = 0; ch < n_ch; ++ch, ++it) {
                const int stage = it % n_stages;
                const uint32_t par = (it / n_stages) & 1;
                mbar_wait(&full[stage], par);
#pragma unroll
                for (int s2 = 0; s2 < kGcCH / 2048; ++s2) {
                    const int cl = (s2 * kGcWarps + slice) * 256 + lane * 8;   // this lane's 8 columns inside the chunk
                    const int c = ch * kGcCH + cl;
                    if (c < cols) {
                        const float4 xa = *reinterpret_cast<const float4*>(xs + c);
                        const float4 xb = *reinterpret_cast<const float4*>(xs + c + 4);
                        const unsigned char* wcol = gc_smem + (size_t)stage * kGcStage + cl * 2;
#pragma unroll
                        for (int r = 0; r < kRowsPer; ++r) {
                            // rows past the CTA's range were not copied: their slots hold stale weights, results unused
                            const uint4 v = *reinterpret_cast<const uint4*>(wcol + (rbase + r) * (kGcCH * 2));
                            float wf[8];
                            unpack8(v, wf);
                            float a0 = fmaf(wf[0], xa.x, acc[r]), a1 = wf[1] * xa.y;
                            a0 = fmaf(wf[2], xa.z, a0); a1 = fmaf(wf[3], xa.w, a1);
                            a0 = fmaf(wf[4], xb.x, a0); a1 = fmaf(wf[5], xb.y, a1);
                            a0 = fmaf(wf[6], xb.z, a0); a1 = fmaf(wf[7], xb.w, a1);
                            acc[r] = a0 + a1;
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
            }
            // rows of the group: lanes -> warp (shuffles), warps -> row (fixed order in shared memory)
            float* part = gpart + (grp & 1) * (kGcWarps * kGcWarps);
#pragma unroll
            for (int r = 0; r < kRowsPer; ++r) {
                const float y = warp_sum(acc[r]);
                if (lane == 0) part[slice * kGcWarps + rbase + r] = y;
            }
            named_bar_sync(1, kC);
            if (tid < kGcWarps && row0 + tid < r_end) {
                float y = 0.f;
#pragma unroll
                for (int w = 0; w < kGcWarps; ++w) y += part[w * kGcWarps + tid];
                const int row = row0 + tid;
                float o = y;
                if (f.epilogue == AF_EPI_GELU_RESIDUAL)
                    o = __ldcg(f.res + row) + 0.5f * y * (1.0f + erff(y * 0.70710678118654752440f));
                else if (f.epilogue == AF_EPI_RESIDUAL)
                    o = __ldcg(f.res + row) + y;
                f.out[row] = o;
            }
        }
        // ---- publish the phase: every warp's rows are written ----
        if (p + 1 < gp.n_phases) {
            named_bar_sync(1, kC);
            if (tid == 0) {
                __threadfence();
                atomicAdd(gp.phase_done + p, 1);
            }
        }
    }
}

}  // namespace af
