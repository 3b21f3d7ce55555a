// af_forward.cuh -- the merged-path forward of ONE token (model.py:367-371 on the Llama block) as ONE persistent
// launch over all layers, driven by a device-side phase table:
//
//     q|k|v(0)  [ attention(l)  o(l)  gate|up(l)  down(l)  q|k|v(l+1) ]  l = 0 .. L-1   (the last q|k|v is the lm_head)
//
// af_gemv_chain (af_gemv_chain.cuh) runs the four projections between two attentions as one launch; what is left
// per layer is the hand-over around the attention kernel: the chained launch drains, the attention's CTAs become
// resident, run, retire, the next chained launch's CTAs become resident, refill their rings -- 14 us of an 88 us
// layer at Llama-2-7B shapes with 1024 cached positions (16 % of the adapter-free decode).  Here the CTAs never leave:
//   * the phase table lives in global memory (one 96-byte record per phase, copied to shared memory while the CTA
//     waits at the phase barrier), so a launch is any number of phases -- 1 + 6 L for a whole forward;
//   * the producer warps stream the weights of every GEMV phase through one ring and run ahead across the attention
//     phases, which have no weights: the ring is full when the consumers come back from an attention;
//   * the attention is two phases of the same kernel: partials -- a team of 8 consumer warps takes one (head, 64-position
//     chunk), one position per warp and step, merges its warps through shared memory and writes (max, sum, acc[hd]);
//     combine -- one thread per output element folds the chunks of its head.  RoPE, the KV append and the use of the
//     new position's own rounded k / v are those of attn_decode2_kernel (af_llama.cuh).
// Arithmetic contract per GEMV phase: that of af_gemv_chain / af_gemv_fused (a row is summed by one warp slice
// order, f32); attention: f32 online softmax, bf16 cache -- the split into chunks differs from the standalone
// kernels', so outputs agree with them to f32 round-off, not bit for bit.
#pragma once

#include "af_gemv_chain.cuh"

namespace af {

constexpr int kFwGemv = 0, kFwAttnPartial = 1, kFwAttnCombine = 2;
constexpr int kFwTeamWarps = 8;                 // warps of a team = positions of a chunk in flight
constexpr int kFwChunk = 64;                    // positions per (head, chunk) work item
constexpr int kFwTeams = kGcCons / kFwTeamWarps;
static_assert(kGcCons % kFwTeamWarps == 0 && kFwTeams >= 1, "consumer warps form whole teams");

struct FwPhase {               // mirrors af_fw_phase (include/adafuse_b200.h)
    const __nv_bfloat16* w;    // GEMV: rows x cols bf16, pitch ld
    const float* x;            // GEMV: input vector; attention partials: q | k | v of the new token (f32)
    float* out;                // GEMV: rows outputs; attention combine: n_heads * head_dim outputs
    const float* res;
    const float* norm_w;
    __nv_bfloat16* k_cache;    // attention: this layer's caches [n_kv][max_seq][head_dim]
    __nv_bfloat16* v_cache;
    long long ld;
    int rows, cols;
    float eps;
    int prologue, epilogue, kind;
};

struct FwParams {
    const FwPhase* table;      // [n_phases], device memory
    int n_phases;
    int* phase_done;           // [n_phases], zeroed by the caller
    int n_stages;
    int pdl;
    int* err_flag;
    // attention geometry, common to all layers
    const float* cos_t;
    const float* sin_t;
    const int* pos_dev;
    int n_heads, n_kv, head_dim, max_seq;
    float scale;
    float* ws;                 // [n_heads][ceil(max_seq / 64)][head_dim + 2] partials
};

// ---- attention partials of one phase: every team loops over its (head, chunk) items ----
template <int HD>
__device__ __noinline__ void fw_attn_partials(const FwPhase& f, const FwParams& A, float* sm_f, int tid, int G) {
    constexpr int EL = HD / 32, half = HD / 2;
    const int lane = tid & 31, warp = tid >> 5;
    const int team = warp / kFwTeamWarps, tw = warp % kFwTeamWarps, tid_t = tid - team * kFwTeamWarps * 32;
    float* m_s = sm_f + team * (kFwTeamWarps * (HD + 2));          // [8] max, [8] sum, [8][HD] acc
    float* l_s = m_s + kFwTeamWarps;
    float* acc_s = l_s + kFwTeamWarps;
    const int pos = __ldcg(A.pos_dev);
    const bool pos_ok = pos >= 0 && pos < A.max_seq;
    const int n_pos = pos_ok ? pos + 1 : 0;
    const int n_chunks = (n_pos + kFwChunk - 1) / kFwChunk, chunks_max = (A.max_seq + kFwChunk - 1) / kFwChunk;
    const int n_items = A.n_heads * n_chunks;
    const int group = A.n_heads / A.n_kv;
    const int rounds = (n_items + kFwTeams * G - 1) / (kFwTeams * G);
    for (int rd = 0; rd < rounds; ++rd) {
        const int item = (rd * G + (int)blockIdx.x) * kFwTeams + team;
        const bool valid = item < n_items;
        float m = -INFINITY, l = 0.f, acc[EL];
#pragma unroll
        for (int e = 0; e < EL; ++e) acc[e] = 0.f;
        int h = 0, j = 0;
        if (valid) {
            h = item / n_chunks;
            j = item % n_chunks;
            const int kvh = h / group;
            const int t0 = j * kFwChunk, t1 = min(n_pos, t0 + kFwChunk);
            const __nv_bfloat16* kbase = f.k_cache + (long long)kvh * A.max_seq * HD;
            const __nv_bfloat16* vbase = f.v_cache + (long long)kvh * A.max_seq * HD;
            // this warp's positions: t0 + tw, + 8, ... (at most 8); their K / V rows first -- they depend on nothing
            constexpr int kPer = kFwChunk / kFwTeamWarps;
            float kf[kPer][EL], vf[kPer][EL];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int t = t0 + tw + u * kFwTeamWarps;
                if (t < t1 && t != pos) {
                    load_bf16_vec<EL>(kbase + (long long)t * HD + lane * EL, kf[u]);
                    load_bf16_vec<EL>(vbase + (long long)t * HD + lane * EL, vf[u]);
                } else {
#pragma unroll
                    for (int e = 0; e < EL; ++e) kf[u][e] = vf[u][e] = 0.f;
                }
            }
            // q of head h with RoPE (rotate-half: dim i pairs with i + half; a lane's partner is lane ^ 16)
            float qv[EL], cs[EL], sn[EL];
#pragma unroll
            for (int e = 0; e < EL; ++e) {
                qv[e] = __ldcg(f.x + (long long)h * HD + lane * EL + e);
                const int i = (lane & 15) * EL + e;
                cs[e] = __ldg(A.cos_t + (long long)pos * half + i);
                sn[e] = __ldg(A.sin_t + (long long)pos * half + i);
            }
            float qr[EL];
#pragma unroll
            for (int e = 0; e < EL; ++e) {
                const float pq = __shfl_xor_sync(0xffffffffu, qv[e], 16);
                qr[e] = (lane < 16 ? qv[e] * cs[e] - pq * sn[e] : qv[e] * cs[e] + pq * sn[e]) * A.scale;
            }
            if (pos >= t0 && pos < t1) {   // the chunk holds the new position: its k / v come from the new token, rounded as the cache stores them
                float kn[EL], vn[EL];
#pragma unroll
                for (int e = 0; e < EL; ++e) {
                    const float kx = __ldcg(f.x + (long long)(A.n_heads + kvh) * HD + lane * EL + e);
                    const float pk = __shfl_xor_sync(0xffffffffu, kx, 16);
                    kn[e] = __bfloat162float(__float2bfloat16_rn(lane < 16 ? kx * cs[e] - pk * sn[e] : kx * cs[e] + pk * sn[e]));
                    vn[e] = __bfloat162float(__float2bfloat16_rn(__ldcg(f.x + (long long)(A.n_heads + A.n_kv + kvh) * HD + lane * EL + e)));
                }
                if (h % group == 0 && tw == 0) {   // one warp per kv head appends to the cache
#pragma unroll
                    for (int e = 0; e < EL; ++e) {
                        f.k_cache[((long long)kvh * A.max_seq + pos) * HD + lane * EL + e] = __float2bfloat16_rn(kn[e]);
                        f.v_cache[((long long)kvh * A.max_seq + pos) * HD + lane * EL + e] = __float2bfloat16_rn(vn[e]);
                    }
                }
#pragma unroll
                for (int u = 0; u < kPer; ++u)
                    if (t0 + tw + u * kFwTeamWarps == pos) {
#pragma unroll
                        for (int e = 0; e < EL; ++e) {
                            kf[u][e] = kn[e];
                            vf[u][e] = vn[e];
                        }
                    }
            }
            float dot[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                float d = 0.f;
#pragma unroll
                for (int e = 0; e < EL; ++e) d = fmaf(qr[e], kf[u][e], d);
                dot[u] = d;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int u = 0; u < kPer; ++u) dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], o);
#pragma unroll
            for (int u = 0; u < kPer; ++u)
                if (t0 + tw + u * kFwTeamWarps < t1) m = fmaxf(m, dot[u]);
#pragma unroll
            for (int u = 0; u < kPer; ++u)
                if (t0 + tw + u * kFwTeamWarps < t1) {   // warp-uniform
                    const float pw = expf(dot[u] - m);
                    l += pw;
#pragma unroll
                    for (int e = 0; e < EL; ++e) acc[e] = fmaf(pw, vf[u][e], acc[e]);
                }
        }
        if (lane == 0) {
            m_s[tw] = m;
            l_s[tw] = l;
        }
#pragma unroll
        for (int e = 0; e < EL; ++e) acc_s[tw * HD + lane * EL + e] = acc[e];
        named_bar_sync(2 + team, kFwTeamWarps * 32);
        if (valid) {   // merge the team's warps: element tid_t of the chunk's un-normalised output
            float mm = -INFINITY;
#pragma unroll
            for (int wv = 0; wv < kFwTeamWarps; ++wv) mm = fmaxf(mm, m_s[wv]);
            float* my = A.ws + ((long long)h * chunks_max + j) * (HD + 2);
            if (tid_t < HD) {
                float o = 0.f;
#pragma unroll
                for (int wv = 0; wv < kFwTeamWarps; ++wv)
                    if (m_s[wv] != -INFINITY) o += acc_s[wv * HD + tid_t] * expf(m_s[wv] - mm);
                my[2 + tid_t] = o;
            }
            if (tid_t == 0) {
                float ll = 0.f;
#pragma unroll
                for (int wv = 0; wv < kFwTeamWarps; ++wv) ll += (m_s[wv] == -INFINITY) ? 0.f : l_s[wv] * expf(m_s[wv] - mm);
                my[0] = mm;
                my[1] = ll;
            }
        }
        named_bar_sync(2 + team, kFwTeamWarps * 32);   // the team's shared memory is free for its next item
    }
}

// ---- attention combine: one thread per output element folds the chunks of its head ----
template <int HD>
__device__ __noinline__ void fw_attn_combine(const FwPhase& f, const FwParams& A, int tid, int G, int n_threads) {
    const int pos = __ldcg(A.pos_dev);
    if (pos < 0 || pos >= A.max_seq) return;
    const int n_chunks = (pos + kFwChunk) / kFwChunk, chunks_max = (A.max_seq + kFwChunk - 1) / kFwChunk;
    const int total = A.n_heads * HD;
    for (int e = (int)blockIdx.x * n_threads + tid; e < total; e += G * n_threads) {
        const int h = e / HD, i = e % HD;
        const float* hp = A.ws + (long long)h * chunks_max * (HD + 2);
        // batches of 16 chunks, every load of a batch issued before the first use: two L2 round trips per batch
        // instead of one per chunk (a run-time-bounded loop of load -> use serialises them: 17 chunks were 12 us)
        constexpr int kB = 16;
        float gm = -INFINITY;
        for (int c0 = 0; c0 < n_chunks; c0 += kB) {
            float pm[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) pm[u] = c0 + u < n_chunks ? __ldcg(hp + (long long)(c0 + u) * (HD + 2)) : -INFINITY;
#pragma unroll
            for (int u = 0; u < kB; ++u) gm = fmaxf(gm, pm[u]);
        }
        float gl = 0.f, o = 0.f;
        for (int c0 = 0; c0 < n_chunks; c0 += kB) {
            float pm[kB], pl[kB], pa[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u) {
                const bool ok = c0 + u < n_chunks;
                const float* q = hp + (long long)(c0 + u) * (HD + 2);
                pm[u] = ok ? __ldcg(q) : -INFINITY;
                pl[u] = ok ? __ldcg(q + 1) : 0.f;
                pa[u] = ok ? __ldcg(q + 2 + i) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kB; ++u)
                if (pm[u] != -INFINITY) {
                    const float w = expf(pm[u] - gm);
                    gl += pl[u] * w;
                    o += pa[u] * w;
                }
        }
        f.out[e] = o / gl;
    }
}

__global__ void __launch_bounds__(kGcThreads, 1) forward_persistent_kernel(const __grid_constant__ FwParams gp) {
    extern __shared__ __align__(128) unsigned char gc_smem[];
    __shared__ uint64_t full[kGcMaxStages], empty[kGcMaxStages];
    __shared__ float redn[kGcCons];
    __shared__ float gpart[2 * kGcWarps * kGcWarps];
    __shared__ FwPhase cur;                 // the phase the consumers are in (copied from the table at its barrier)
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
    auto row_begin = [&](int rows, int c) { return (int)((long long)rows * c / G); };

    if (warp >= kGcCons) {
        // ===================== producers: the weights of every GEMV phase, back to back ==========
        if (lane == 0) {
            const int who = warp - kGcCons;
            const uint32_t base = smem_u32(gc_smem);
            int it = 0;
            for (int p = 0; p < gp.n_phases; ++p) {
                const FwPhase* f = gp.table + p;
                if (__ldg(&f->kind) != kFwGemv) continue;
                const int rows = __ldg(&f->rows), cols = __ldg(&f->cols);
                const long long ld = __ldg(&f->ld);
                const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(__ldg(reinterpret_cast<const unsigned long long*>(&f->w)));
                const int r_begin = row_begin(rows, blockIdx.x), r_end = row_begin(rows, blockIdx.x + 1);
                const int n_ch = (cols + kGcCH - 1) / kGcCH;
                for (int row0 = r_begin; row0 < r_end; row0 += kGcWarps) {
                    const int nrow = min(kGcWarps, r_end - row0);
                    for (int ch = 0; ch < n_ch; ++ch, ++it) {
                        const int stage = it % n_stages;
                        const uint32_t par = (it / n_stages) & 1;
                        const int c0 = ch * kGcCH;
                        const uint32_t bytes = (uint32_t)min(kGcCH, cols - c0) * 2;
                        int mine = 0;
                        for (int r = who; r < nrow; r += kGcProd) ++mine;
                        mbar_wait(&empty[stage], par ^ 1);
                        mbar_expect_tx(&full[stage], bytes * mine);
                        for (int r = who; r < nrow; r += kGcProd)
                            gv_bulk_load(base + stage * kGcStage + r * (kGcCH * 2), w + (long long)(row0 + r) * ld + c0, bytes, &full[stage]);
                    }
                }
            }
        }
        return;
    }

    // ===================== consumers =====================
    constexpr int kC = kGcCons * 32;
    constexpr int kRowsPer = kGcWarps / kGcHalves;
    const int slice = warp % kGcWarps, rbase = (warp / kGcWarps) * kRowsPer;
    if (gp.pdl) {
        pdl_wait();
        if (tid == 0) pdl_launch_dependents();
    }
    int it = 0;
    for (int p = 0; p < gp.n_phases; ++p) {
        // the phase record: static, so it is fetched before (not after) the wait for the previous phase
        named_bar_sync(1, kC);   // everyone is done with the previous record
        if (tid < (int)(sizeof(FwPhase) / 4)) reinterpret_cast<int*>(&cur)[tid] = __ldg(reinterpret_cast<const int*>(gp.table + p) + tid);
        if (p > 0) {
            if (tid == 0) {
                const long long t0 = clock64();
                int seen;
                unsigned spins = 0;
                do {
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(gp.phase_done + p - 1) : "memory");
                    if (seen >= G) break;
                    if ((++spins & 1023u) == 0 && gp.err_flag && *reinterpret_cast<volatile int*>(gp.err_flag) == AF_ECUDA) break;
                    if (clock64() - t0 > (1ll << 32)) {   // ~2 s: never hang the device on a lost CTA
                        if (gp.err_flag) atomicExch(gp.err_flag, AF_ECUDA);
                        break;
                    }
                } while (true);
            }
        }
        named_bar_sync(1, kC);
        const FwPhase& f = cur;
        if (f.kind == kFwAttnPartial) {
            if (gp.head_dim == 128) fw_attn_partials<128>(f, gp, xs, tid, G);
            else fw_attn_partials<64>(f, gp, xs, tid, G);
        } else if (f.kind == kFwAttnCombine) {
            if (gp.head_dim == 128) fw_attn_combine<128>(f, gp, tid, G, kC);
            else fw_attn_combine<64>(f, gp, tid, G, kC);
        } else {
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
            // ---- this CTA's rows in groups of 8 (the arithmetic of gemv_chain_kernel, unchanged) ----
            const int r_begin = row_begin(f.rows, blockIdx.x), r_end = row_begin(f.rows, blockIdx.x + 1);
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
                        const int cl = (s2 * kGcWarps + slice) * 256 + lane * 8;
                        const int c = ch * kGcCH + cl;
                        if (c < cols) {
                            const float4 xa = *reinterpret_cast<const float4*>(xs + c);
                            const float4 xb = *reinterpret_cast<const float4*>(xs + c + 4);
                            const unsigned char* wcol = gc_smem + (size_t)stage * kGcStage + cl * 2;
#pragma unroll
                            for (int r = 0; r < kRowsPer; ++r) {
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
        }
        // ---- publish the phase: every warp's outputs are written ----
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
