// af_switch.cuh -- the fused switching kernel.
//
// Replaces, per token, adapters.py:188-211 `concat_gated` x L, adapters.py:214-233
// `build_switch` x L and adapters.py:236-258 `merge_all` -> linalg.py:306-346 `sgmm`
// with ONE persistent launch over every adapted matrix:
//
//     W <- bf16( W + sum_{b in cur} g_b * B_b A_b - sum_{b in prev} g'_b * B_b A_b )
//
// Nothing is concatenated: a per-launch block list (expert id, signed f32 weight) selects
// rows of the resident expert bank, and the gate is folded into the DOWN rows while they are
// staged in shared memory (adapters.py:202).
//
// Two kernels:
//   switch_tma_kernel   bf16 targets whose rows are 16-byte aligned: W tiles move through a
//                       4-stage TMA ring (load -> update in smem -> TMA store in place), one
//                       producer warp + 8 consumer warps, grid = #SMs, static unit schedule.
//   switch_any_kernel   any shape / alignment / dtype (f32 "single" targets, odd sizes);
//                       also the in-GPU cross-check of the fast kernel.
#pragma once

#include <cuda.h>

#include "af_common.cuh"

namespace af {

constexpr int kTM = 64;          // tile rows
constexpr int kTN = 256;         // tile cols (one TMA box row = 512 B of bf16)
constexpr int kStages = 4;       // W tiles in flight per SM (4 x 32 KB)
constexpr int kSlabRanks = 32;   // ranks staged per pass (f32 slabs: down 32 KB, up 8/16 KB)
constexpr int kConsumers = 256;  // 8 consumer warps
constexpr int kMaxBlocks = 2 * AF_MAX_K;

struct SegDev {
    void* target;
    const void* pristine;
    const void* down;
    const void* up;
    int d_out, d_in, rank, n_experts;
    long long ld_target, ld_down, ld_up, down_estride, up_estride;
};

// One work unit: rows [row0, row0+rows) x cols [col0, col0+kTN) of segment `seg`.
struct UnitDev {
    int seg, row0, rows, col0;
    int phase;  // chained switch + GEMV launches: which projection of the chain the unit belongs to
    int slot;   // ... and the segment's position in the chain's segment list (shared-memory descriptor cache)
};

struct Plan {
    int n_blocks;
    int expert[kMaxBlocks];
    float weight[kMaxBlocks];  // signed, scale folded in
    int negate[kMaxBlocks];    // EXACT mode: weight is the positive gate, negate after folding
};

struct SwitchParams {
    const SegDev* segs;
    const UnitDev* units;
    const CUtensorMap* tmaps_src;  // per segment: where tiles are read from (live or pristine)
    const CUtensorMap* tmaps_dst;  // per segment: the live matrix
    int n_units;
    int from_pristine;
    const af_decision* prev_dev;
    const af_decision* cur_dev;
    int use_dev;  // 1: build the plan on device from prev_dev/cur_dev; 0: host_plan
    float scale;
    int n_experts_limit;  // smallest bank over the table: ids outside [0, limit) are rejected
    int max_blocks;       // block-list capacity this launch was sized for (kernel variant, smem)
    int* err_flag;        // device word: set to AF_EINDEX / AF_EVALUE when a device decision is unusable
    const Plan* plan_dev; // block list built once per token by plan_build_kernel (af_plan_build); NULL: build it here
    Plan host_plan;
};

// Validate the device-built plan against what the host sized the launch for.  A decision that
// names an expert outside the bank (adapters.py:199-200 -> IndexError) or carries more blocks
// than the launch can hold makes the whole launch a no-op and raises the table's error flag.
__device__ __forceinline__ bool plan_usable(const SwitchParams& p, const Plan& plan, const af_decision* prev,
                                            const af_decision* cur) {
    int bad = 0;
    if (p.use_dev) {
        const af_decision* d2[2] = {p.from_pristine ? nullptr : prev, cur};
        for (int s = 0; s < 2; ++s) {
            if (!d2[s]) continue;
            if (d2[s]->k < 0 || d2[s]->k > AF_MAX_K) bad = AF_EVALUE;
            else
                for (int j = 0; j < d2[s]->k; ++j)
                    if (d2[s]->ids[j] < 0 || d2[s]->ids[j] >= p.n_experts_limit) bad = AF_EINDEX;
        }
    }
    if (!bad && plan.n_blocks > p.max_blocks) bad = AF_EVALUE;
    if (bad && p.err_flag) atomicExch(p.err_flag, bad);
    return bad == 0;
}

// Build the block list from two decisions (either may be null == empty concat).
// exact == true : reference order, prev blocks then cur blocks, no collapsing
//                 (adapters.py:230-231); weight = gate, negate marks prev.
// exact == false: an expert present on both sides contributes ONE block with weight
//                 (g_new - g_old); blocks whose weight is exactly 0 vanish, so an unchanged
//                 decision makes the launch a no-op.
__host__ __device__ inline void build_plan(Plan& plan, const af_decision* prev, const af_decision* cur,
                                           float scale, bool exact, int n_experts_limit) {
    plan.n_blocks = 0;
    int kp = prev ? prev->k : 0;
    int kc = cur ? cur->k : 0;
    kp = kp < 0 ? 0 : (kp > AF_MAX_K ? AF_MAX_K : kp);
    kc = kc < 0 ? 0 : (kc > AF_MAX_K ? AF_MAX_K : kc);
    if (exact) {
        for (int j = 0; j < kp && plan.n_blocks < kMaxBlocks; ++j) {
            int e = prev->ids[j];
            if (e < 0 || e >= n_experts_limit) continue;
            plan.expert[plan.n_blocks] = e;
            plan.weight[plan.n_blocks] = prev->weights[j] * scale;
            plan.negate[plan.n_blocks] = 1;
            ++plan.n_blocks;
        }
        for (int j = 0; j < kc && plan.n_blocks < kMaxBlocks; ++j) {
            int e = cur->ids[j];
            if (e < 0 || e >= n_experts_limit) continue;
            plan.expert[plan.n_blocks] = e;
            plan.weight[plan.n_blocks] = cur->weights[j] * scale;
            plan.negate[plan.n_blocks] = 0;
            ++plan.n_blocks;
        }
        return;
    }
    // Net weight per distinct expert, in order of first appearance (cur, then prev):
    //   w_e = (sum of e's gates in cur - sum of e's gates in prev) * scale ;  w_e == 0 -> no block.
    // (Duplicates inside one decision are summed, wherever the first occurrence netted to.)
    for (int side = 0; side < 2; ++side) {
        const af_decision* d = side == 0 ? cur : prev;
        const int kd = side == 0 ? kc : kp;
        for (int j = 0; j < kd; ++j) {
            const int e = d->ids[j];
            if (e < 0 || e >= n_experts_limit) continue;
            bool seen = false;
            for (int i = 0; i < j; ++i)
                if (d->ids[i] == e) seen = true;
            if (side == 1)
                for (int i = 0; i < kc; ++i)
                    if (cur->ids[i] == e) seen = true;
            if (seen) continue;
            float w = 0.0f;
            for (int i = 0; i < kc; ++i)
                if (cur->ids[i] == e) w += cur->weights[i];
            for (int i = 0; i < kp; ++i)
                if (prev->ids[i] == e) w -= prev->weights[i];
            w *= scale;
            if (w == 0.0f || plan.n_blocks >= kMaxBlocks) continue;
            plan.expert[plan.n_blocks] = e;
            plan.weight[plan.n_blocks] = w;
            plan.negate[plan.n_blocks] = 0;
            ++plan.n_blocks;
        }
    }
}

// One launch per token (af_plan_build): the block list every switch + GEMV launch of the token
// would otherwise rebuild from the two decisions at its start (2.6 us of serial work per launch).
__global__ void plan_build_kernel(SwitchParams p, Plan* out) {
    if (threadIdx.x != 0) return;
    Plan plan;
    build_plan(plan, p.from_pristine ? nullptr : p.prev_dev, p.cur_dev, p.scale, false, p.n_experts_limit);
    if (!plan_usable(p, plan, p.prev_dev, p.cur_dev)) plan.n_blocks = -1;
    *out = plan;
}

// ---------------------------------------------------------------------------
// Slab staging shared by both kernels.
//   down slab: f32 [ranks][kTN], gate folded in (adapters.py:202), prev blocks negated
//              (adapters.py:230); columns past d_in are 0.
//   up slab  : f32 [ranks][kTM] (rank-major so one thread's 8 rows are contiguous).
// Slab row q (global rank index) belongs to block q / rank, in-block row q % rank.
// ---------------------------------------------------------------------------

template <typename FT, bool EXACT>
__device__ __forceinline__ void fill_down_slab(float* __restrict__ slab, const SegDev& sg, const Plan& plan,
                                               int q0, int q1, int col0, int tid, int nthreads) {
    const FT* base = reinterpret_cast<const FT*>(sg.down);
    const int r = sg.rank;
    const bool vec_ok = sizeof(FT) == 2 && (sg.ld_down % 8 == 0) && (sg.down_estride % 8 == 0) &&
                        ((reinterpret_cast<uintptr_t>(base) & 15) == 0) && (sg.d_in % 8 == 0);
    if (vec_ok) {
        // 16-byte (8 x bf16) loads; a chunk is entirely inside or outside the matrix.
        const int chunks_per_row = kTN / 8;
        const int total = (q1 - q0) * chunks_per_row;
        for (int i = tid; i < total; i += nthreads) {
            const int ql = i / chunks_per_row;
            const int c = (i % chunks_per_row) * 8;
            const int q = q0 + ql;
            const int b = q / r, qr = q % r;
            float4 lo = make_float4(0.f, 0.f, 0.f, 0.f), hi = lo;
            if (col0 + c < sg.d_in) {
                const FT* src = base + (long long)plan.expert[b] * sg.down_estride + (long long)qr * sg.ld_down + col0 + c;
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(src));
                const float w = plan.weight[b];
                float f[8] = {bf16lo_to_f32(v.x), bf16hi_to_f32(v.x), bf16lo_to_f32(v.y), bf16hi_to_f32(v.y),
                              bf16lo_to_f32(v.z), bf16hi_to_f32(v.z), bf16lo_to_f32(v.w), bf16hi_to_f32(v.w)};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    f[j] = __fmul_rn(w, f[j]);
                    if (EXACT && plan.negate[b]) f[j] = -f[j];
                }
                lo = make_float4(f[0], f[1], f[2], f[3]);
                hi = make_float4(f[4], f[5], f[6], f[7]);
            }
            float4* dst = reinterpret_cast<float4*>(slab + ql * kTN + c);
            dst[0] = lo;
            dst[1] = hi;
        }
    } else {
        const int total = (q1 - q0) * kTN;
        for (int i = tid; i < total; i += nthreads) {
            const int ql = i / kTN, c = i % kTN;
            const int q = q0 + ql;
            const int b = q / r, qr = q % r;
            float v = 0.f;
            if (col0 + c < sg.d_in) {
                const FT* src = base + (long long)plan.expert[b] * sg.down_estride + (long long)qr * sg.ld_down + col0 + c;
                v = __fmul_rn(plan.weight[b], load_as_f32<FT>(src));
                if (EXACT && plan.negate[b]) v = -v;
            }
            slab[ql * kTN + c] = v;
        }
    }
}

template <typename FT>
__device__ __forceinline__ float load_up_elem(const SegDev& sg, const Plan& plan, int q, int row) {
    const int b = q / sg.rank, qr = q % sg.rank;
    const FT* src = reinterpret_cast<const FT*>(sg.up) + (long long)plan.expert[b] * sg.up_estride +
                    (long long)row * sg.ld_up + qr;
    return load_as_f32<FT>(src);
}

// ---------------------------------------------------------------------------
// Fast path: TMA-staged bf16 tiles.
// ---------------------------------------------------------------------------

struct alignas(128) SwitchSmem {
    // W tile ring: kStages x [kTM][kTN] bf16, dense (TMA box, no swizzle)
    __nv_bfloat16 w[kStages][kTM * kTN];
    float down[kSlabRanks * kTN];   // 32 KB
    float up2[kSlabRanks * kTM * 2];  // 16 KB: (u,u) pairs when F2, else first half used
    uint64_t full[kStages];
    uint64_t empty[kStages];
    Plan plan;
};

// Accumulators are kept as float2 pairs along the column direction so the packed
// fma.rn.f32x2 path (F2) maps onto 64-bit register pairs; A(i,j) is the scalar view.
#define AF_ACC(i, j) (((j) & 1) ? acc[i][(j) >> 1].y : acc[i][(j) >> 1].x)

template <bool EXACT, bool F2>
__device__ __forceinline__ void tile_update(SwitchSmem& sm, int stage, int n_ranks, bool first_pass,
                                            bool last_pass, float2 (&acc)[8][4], int tx, int ty) {
    __nv_bfloat16* wt = sm.w[stage];
    // EXACT starts from W and applies every rank in order; FMA accumulates the delta from 0.
    if (first_pass) {
        if (EXACT) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint4 v = *reinterpret_cast<const uint4*>(wt + (ty * 8 + i) * kTN + tx * 8);
                acc[i][0] = make_float2(bf16lo_to_f32(v.x), bf16hi_to_f32(v.x));
                acc[i][1] = make_float2(bf16lo_to_f32(v.y), bf16hi_to_f32(v.y));
                acc[i][2] = make_float2(bf16lo_to_f32(v.z), bf16hi_to_f32(v.z));
                acc[i][3] = make_float2(bf16lo_to_f32(v.w), bf16hi_to_f32(v.w));
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
        }
    }
    if (F2 && !EXACT) {
        const float2* up2 = reinterpret_cast<const float2*>(sm.up2);
#pragma unroll 2
        for (int q = 0; q < n_ranks; ++q) {
            const float4 d0 = *reinterpret_cast<const float4*>(sm.down + q * kTN + tx * 8);
            const float4 d1 = *reinterpret_cast<const float4*>(sm.down + q * kTN + tx * 8 + 4);
            const float2 dp[4] = {make_float2(d0.x, d0.y), make_float2(d0.z, d0.w), make_float2(d1.x, d1.y),
                                  make_float2(d1.z, d1.w)};
            const float4* urow = reinterpret_cast<const float4*>(up2 + q * kTM + ty * 8);
#pragma unroll
            for (int ih = 0; ih < 4; ++ih) {
                const float4 uu = urow[ih];  // (u_{2ih}, u_{2ih}, u_{2ih+1}, u_{2ih+1})
                const float2 ua = make_float2(uu.x, uu.y), ub = make_float2(uu.z, uu.w);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[2 * ih][j] = ffma2(ua, dp[j], acc[2 * ih][j]);
                    acc[2 * ih + 1][j] = ffma2(ub, dp[j], acc[2 * ih + 1][j]);
                }
            }
        }
    } else {
        const float* up = sm.up2;
#pragma unroll 2
        for (int q = 0; q < n_ranks; ++q) {
            const float4 d0 = *reinterpret_cast<const float4*>(sm.down + q * kTN + tx * 8);
            const float4 d1 = *reinterpret_cast<const float4*>(sm.down + q * kTN + tx * 8 + 4);
            const float d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
            const float4 u0 = *reinterpret_cast<const float4*>(up + q * kTM + ty * 8);
            const float4 u1 = *reinterpret_cast<const float4*>(up + q * kTM + ty * 8 + 4);
            const float u[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (EXACT)
                        AF_ACC(i, j) = __fadd_rn(AF_ACC(i, j), __fmul_rn(u[i], d[j]));  // linalg.py:338-341
                    else
                        AF_ACC(i, j) = fmaf(u[i], d[j], AF_ACC(i, j));
                }
        }
    }
    if (last_pass) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint4* p = reinterpret_cast<uint4*>(wt + (ty * 8 + i) * kTN + tx * 8);
            float2 o[4];
            if (EXACT) {
#pragma unroll
                for (int j = 0; j < 4; ++j) o[j] = acc[i][j];
            } else {
                const uint4 v = *p;
                o[0] = make_float2(bf16lo_to_f32(v.x) + acc[i][0].x, bf16hi_to_f32(v.x) + acc[i][0].y);
                o[1] = make_float2(bf16lo_to_f32(v.y) + acc[i][1].x, bf16hi_to_f32(v.y) + acc[i][1].y);
                o[2] = make_float2(bf16lo_to_f32(v.z) + acc[i][2].x, bf16hi_to_f32(v.z) + acc[i][2].y);
                o[3] = make_float2(bf16lo_to_f32(v.w) + acc[i][3].x, bf16hi_to_f32(v.w) + acc[i][3].y);
            }
            uint4 w;
            w.x = pack_bf16x2(o[0].x, o[0].y);
            w.y = pack_bf16x2(o[1].x, o[1].y);
            w.z = pack_bf16x2(o[2].x, o[2].y);
            w.w = pack_bf16x2(o[3].x, o[3].y);
            *p = w;
        }
    }
}

// Tile iterator over this CTA's static schedule: units blockIdx.x, +gridDim.x, ...; inside a
// unit, kTM-row tiles top to bottom.  Producer and consumers walk the same sequence.
template <int STEP>
struct TileIterT {
    int u, m0, row_end;
    UnitDev un;
    __device__ __forceinline__ bool valid(const SwitchParams& p) const { return u < p.n_units; }
    // A unit with rows == 0 is padding of a per-CTA list (group schedules, af_group_create):
    // a CTA's list has no holes, so the first empty unit ends its walk.
    __device__ __forceinline__ void load_unit(const SwitchParams& p) {
        if (u < p.n_units) {
            un = p.units[u];
            m0 = un.row0;
            row_end = un.row0 + un.rows;
            if (un.rows <= 0) u = p.n_units;
        }
    }
    __device__ __forceinline__ void init(const SwitchParams& p) {
        u = blockIdx.x;
        load_unit(p);
    }
    // returns true when the step crossed into a new unit
    __device__ __forceinline__ bool next(const SwitchParams& p) {
        m0 += STEP;
        if (m0 < row_end) return false;
        u += gridDim.x;
        load_unit(p);
        return true;
    }
};
using TileIter = TileIterT<kTM>;

// Vectorised UP staging: one 16-byte chunk = 8 consecutive ranks of one (row, block).
// Eligible when every block's rows are 16-byte aligned and rank % 8 == 0 (bf16 banks).
template <typename FT>
__device__ __forceinline__ bool up_vec_ok(const SegDev& sg) {
    return sizeof(FT) == 2 && sg.rank % 8 == 0 && sg.ld_up % 8 == 0 && sg.up_estride % 8 == 0 &&
           (reinterpret_cast<uintptr_t>(sg.up) & 15) == 0;
}

template <typename FT>
__device__ __forceinline__ uint4 up_vec_load(const SegDev& sg, const Plan& plan, int chunk, int m0) {
    // chunk -> (rank group g of 8 ranks, row); row fastest so a warp reads 32 consecutive rows
    const int row = chunk % kTM, g = chunk / kTM;
    const int q = g * 8;
    const int b = q / sg.rank, qr = q % sg.rank;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (m0 + row < sg.d_out) {
        const FT* src = reinterpret_cast<const FT*>(sg.up) + (long long)plan.expert[b] * sg.up_estride +
                        (long long)(m0 + row) * sg.ld_up + qr;
        v = __ldg(reinterpret_cast<const uint4*>(src));
    }
    return v;
}

template <bool PAIRS>
__device__ __forceinline__ void up_vec_store(float* up2, int chunk, uint4 v) {
    const int row = chunk % kTM, g = chunk / kTM;
    const float f[8] = {bf16lo_to_f32(v.x), bf16hi_to_f32(v.x), bf16lo_to_f32(v.y), bf16hi_to_f32(v.y),
                        bf16lo_to_f32(v.z), bf16hi_to_f32(v.z), bf16lo_to_f32(v.w), bf16hi_to_f32(v.w)};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (PAIRS)
            reinterpret_cast<float2*>(up2)[(g * 8 + j) * kTM + row] = make_float2(f[j], f[j]);
        else
            up2[(g * 8 + j) * kTM + row] = f[j];
    }
}

template <typename FT, bool EXACT, bool F2>
__global__ void __launch_bounds__(kConsumers + 32, 1) switch_tma_kernel(const __grid_constant__ SwitchParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SwitchSmem& sm = *reinterpret_cast<SwitchSmem*>(smem_raw);
    const int tid = threadIdx.x;
    constexpr bool PAIRS = F2 && !EXACT;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        fence_mbar_init();
        if (p.use_dev) {
            build_plan(sm.plan, p.from_pristine ? nullptr : p.prev_dev, p.cur_dev, p.scale, EXACT,
                       p.n_experts_limit);
        } else {
            sm.plan = p.host_plan;
        }
        if (!plan_usable(p, sm.plan, p.prev_dev, p.cur_dev)) sm.plan.n_blocks = -1;
    }
    __syncthreads();
    const int n_blocks = sm.plan.n_blocks;
    if (n_blocks < 0) return;                       // unusable decision: flagged, nothing touched
    if (n_blocks == 0 && !p.from_pristine) return;  // unchanged decision: nothing to move

    if (tid >= kConsumers) {
        // ===================== producer warp: TMA loads of W tiles =====================
        if (tid == kConsumers) {
            TileIter ti;
            ti.init(p);
            for (int it = 0; ti.valid(p); ++it) {
                const int stage = it % kStages;
                const uint32_t ph = (it / kStages) & 1;
                mbar_wait(&sm.empty[stage], ph ^ 1);
                mbar_expect_tx(&sm.full[stage], kTM * kTN * 2);
                tma_load_2d(sm.w[stage], p.tmaps_src + ti.un.seg, ti.un.col0, ti.m0, &sm.full[stage]);
                ti.next(p);
            }
        }
        return;
    }

    // ============================ consumer warps ====================================
    const int tx = tid & 31, ty = tid >> 5;
    float2 acc[8][4];
    int prev_stage = -1;
    TileIter ti;
    ti.init(p);
    bool new_unit = true;
    SegDev sg;
    int S = 0, n_pass = 1;
    bool vec = false;      // UP staged with prefetched 16-byte chunks (single pass, <= 1 chunk/thread)
    bool have_pref = false;
    uint4 pref = make_uint4(0u, 0u, 0u, 0u);
    for (int it = 0; ti.valid(p); ++it) {
        const int stage = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        if (new_unit) {
            sg = p.segs[ti.un.seg];
            S = n_blocks * sg.rank;
            n_pass = (S + kSlabRanks - 1) / kSlabRanks;
            vec = up_vec_ok<FT>(sg) && n_pass == 1 && S > 0;
            if (n_pass == 1) {  // the whole gated DOWN strip fits: stage it once per unit
                named_bar_sync(1, kConsumers);
                fill_down_slab<FT, EXACT>(sm.down, sg, sm.plan, 0, S, ti.un.col0, tid, kConsumers);
            }
            if (vec && !have_pref && tid < (S / 8) * kTM) pref = up_vec_load<FT>(sg, sm.plan, tid, ti.m0);
        }
        const int m0 = ti.m0;
        const UnitDev un = ti.un;
        for (int pass = 0; pass < (n_pass > 0 ? n_pass : 1); ++pass) {
            const int q0 = pass * kSlabRanks;
            const int q1 = min(S, q0 + kSlabRanks);
            named_bar_sync(1, kConsumers);  // previous readers of the slabs are done
            if (n_pass > 1) fill_down_slab<FT, EXACT>(sm.down, sg, sm.plan, q0, q1, un.col0, tid, kConsumers);
            if (vec) {
                if (tid < (S / 8) * kTM) up_vec_store<PAIRS>(sm.up2, tid, pref);
            } else {
                // scalar UP staging: f32, rank-major; rows past d_out are 0
                for (int i = tid; i < (q1 - q0) * kTM; i += kConsumers) {
                    const int ql = i / kTM, row = i % kTM;
                    const float v = (m0 + row < sg.d_out) ? load_up_elem<FT>(sg, sm.plan, q0 + ql, m0 + row) : 0.f;
                    if (PAIRS)
                        reinterpret_cast<float2*>(sm.up2)[ql * kTM + row] = make_float2(v, v);
                    else
                        sm.up2[ql * kTM + row] = v;
                }
            }
            named_bar_sync(1, kConsumers);  // slabs visible
            if (pass == 0) {
                // advance the schedule now so the next tile's UP chunk is in flight during the math
                new_unit = ti.next(p);
                have_pref = false;
                if (vec && !new_unit && ti.valid(p)) {
                    if (tid < (S / 8) * kTM) pref = up_vec_load<FT>(sg, sm.plan, tid, ti.m0);
                    have_pref = true;
                }
                mbar_wait(&sm.full[stage], ph);
            }
            tile_update<EXACT, F2>(sm, stage, q1 - q0, pass == 0, pass >= n_pass - 1, acc, tx, ty);
        }
        fence_proxy_async_smem();
        named_bar_sync(2, kConsumers);  // whole tile written back to smem
        if (tid == 0) {
            tma_store_2d(p.tmaps_dst + un.seg, un.col0, m0, sm.w[stage]);
            bulk_commit();
            bulk_wait_read<1>();  // the store issued one tile ago has drained its smem
            if (prev_stage >= 0) mbar_arrive(&sm.empty[prev_stage]);
            prev_stage = stage;
        }
    }
    if (tid == 0) bulk_wait_all<0>();
}

// ---------------------------------------------------------------------------
// General path: any dtype, any shape, any rank total; plain loads/stores, factors read
// straight from global memory (L1/L2 resident).  One CTA per unit; thread t owns column
// col0 + t of the strip and walks the unit's rows.  Also the in-GPU cross-check of the
// fast kernel.
// ---------------------------------------------------------------------------

template <typename WT, typename FT, bool EXACT>
__global__ void __launch_bounds__(kTN) switch_any_kernel(const __grid_constant__ SwitchParams p) {
    __shared__ Plan plan;
    const int tid = threadIdx.x;
    if (tid == 0) {
        if (p.use_dev)
            build_plan(plan, p.from_pristine ? nullptr : p.prev_dev, p.cur_dev, p.scale, EXACT, p.n_experts_limit);
        else
            plan = p.host_plan;
        if (!plan_usable(p, plan, p.prev_dev, p.cur_dev)) plan.n_blocks = -1;
    }
    __syncthreads();
    if (plan.n_blocks < 0) return;
    if (plan.n_blocks == 0 && !p.from_pristine) return;
    for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
        const UnitDev un = p.units[u];
        const SegDev sg = p.segs[un.seg];
        const int col = un.col0 + tid;
        if (col >= sg.d_in) continue;
        WT* tgt = reinterpret_cast<WT*>(sg.target);
        const WT* src = p.from_pristine ? reinterpret_cast<const WT*>(sg.pristine) : tgt;
        const FT* down = reinterpret_cast<const FT*>(sg.down);
        for (int row = un.row0; row < un.row0 + un.rows; ++row) {
            const long long off = (long long)row * sg.ld_target + col;
            float acc = load_as_f32<WT>(src + off);
            float delta = 0.f;
            for (int b = 0; b < plan.n_blocks; ++b) {
                const float w = plan.weight[b];
                const FT* dn = down + (long long)plan.expert[b] * sg.down_estride + col;
                for (int qr = 0; qr < sg.rank; ++qr) {
                    float dq = __fmul_rn(w, load_as_f32<FT>(dn + (long long)qr * sg.ld_down));  // adapters.py:202
                    if (EXACT && plan.negate[b]) dq = -dq;                                      // adapters.py:230
                    const float uq = load_up_elem<FT>(sg, plan, b * sg.rank + qr, row);
                    if (EXACT)
                        acc = __fadd_rn(acc, __fmul_rn(uq, dq));  // linalg.py:338-341
                    else
                        delta = fmaf(uq, dq, delta);
                }
            }
            if (!EXACT) acc += delta;
            store_from_f32<WT>(tgt + off, acc);
        }
    }
}

}  // namespace af
