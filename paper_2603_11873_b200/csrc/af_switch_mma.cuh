// af_switch_mma.cuh -- fused switching kernel, HBM-bound variant.
//
// Same contract as af_switch.cuh (adapters.py:188-258 + linalg.py:306-346 in one persistent
// launch) but the rank-s micro product  D = sum_b g_b * B_b A_b  is issued on the tensor pipe
// (mma.sync m16n8k16, bf16 in, f32 accumulate) so the CUDA cores only do the W + D add and
// the bf16 rounding.  On fp32 FMA the steady switch (s = 2kr = 32) needs 104 TFLOP/s to keep
// up with HBM -- above the FMA peak of the chip; here the math is ~15 % of
// the tile time and the kernel is bound by the W stream.
//
// Gate weights stay f32: the gated DOWN row v = g * a (one f32 multiply, adapters.py:202) is
// split into v = hi + lo + O(2^-17 |v|) with hi, lo bf16, and D = U.hi + U.lo accumulates in
// f32 (products of two bf16 values are exact in f32).
//
// Data movement per 32 x 256 tile of W (one pipeline stage, 16 KB):
//   W   : 4 TMA boxes of 32 rows x 64 cols (128-byte swizzle) global -> smem, updated in place
//         in smem with ldmatrix / stmatrix, then 4 TMA box stores by a dedicated storer warp.
//   UP  : one 1-D bulk copy per block (32 rows x r bf16 are contiguous in the bank).
//   DOWN: gated hi/lo slab [2 * S_pad][256 (+8 pad)] bf16, staged once per unit (column strip);
//         each consumer warp owns 16 columns of the strip and keeps its B fragments of the slab
//         in registers for the whole unit, so the slab is read once per unit, not once per tile.
#pragma once

#include "af_switch.cuh"

namespace af {

#ifndef AF_MR
#define AF_MR 32
#endif
#ifndef AF_WPROD
#define AF_WPROD 1      /* threads (one per warp) issuing the W box loads */
#endif
#ifndef AF_STORERS
#define AF_STORERS 1    /* threads (one per warp) issuing the W box stores */
#endif
constexpr int kMR = AF_MR;                        // tile rows of the tensor path
constexpr int kBoxCols = 64;                      // 128-byte swizzle span in bf16
constexpr int kBoxes = kTN / kBoxCols;            // 4 boxes per tile
constexpr int kBoxBytes = kMR * kBoxCols * 2;     // 4 KB
constexpr int kWStageBytes = kMR * kTN * 2;       // 16 KB
constexpr int kDownPitch = kTN + 8;               // elements; +16 B keeps ldmatrix conflict free
constexpr int kMmaWarps = 16;                     // consumer warps: one n16 column slice each
constexpr int kMmaConsumers = kMmaWarps * 32;     // 512 threads
constexpr int kWProd = AF_WPROD;                  // W-load producer warps
constexpr int kStorers = AF_STORERS;              // storer warps
constexpr int kMmaThreads = kMmaConsumers + 32 * (kWProd + 1 + kStorers);  // + W producers + UP producer + storers
constexpr int kMmaMaxKS = 4;                      // k-steps of 16 ranks: S <= 64
constexpr int kMmaMaxStages = 12;
constexpr int kStoreDepth = 0;                    // tile stores that may still be reading smem
constexpr int kMmaDefaultStages = 10;

template <int KS>
struct MmaLayout {
    static constexpr int s_pad = KS * 16;
    static constexpr int up_stage_bytes = kMR * s_pad * 2;
    static constexpr int down_bytes = 2 * s_pad * kDownPitch * 2;
    static constexpr int fixed = down_bytes + 3 * 8 * 16 + (int)sizeof(Plan) + 1024 /*alignment slack*/ + 256;
    static constexpr int by_smem = (227 * 1024 - fixed) / (kWStageBytes + up_stage_bytes);
    static constexpr int stages = by_smem < kMmaMaxStages ? by_smem : kMmaMaxStages;
    // offsets from the 1024-aligned base
    static constexpr int off_w = 0;
    static constexpr int off_up = off_w + stages * kWStageBytes;
    static constexpr int off_down = off_up + stages * up_stage_bytes;
    static constexpr int off_bar = off_down + down_bytes;          // full[16], computed[16], empty[16]
    static constexpr int off_plan = off_bar + 3 * 8 * 16;
    static constexpr int total = off_plan + (int)sizeof(Plan) + 1024 /*alignment slack*/;
    static_assert(stages >= 3 && total <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void stmatrix_x4(uint32_t addr, const uint32_t (&r)[4]) {
    asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 : "memory");
}
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 1-D bulk copy global -> smem, completes on bar (bytes % 16 == 0, both sides 16-byte aligned).
__device__ __forceinline__ void bulk_load_1d(uint32_t smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d_addr(uint32_t smem_dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_dst), "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d_addr(const void* tmap, int c0, int c1, uint32_t smem_src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap), "r"(c0),
                 "r"(c1), "r"(smem_src)
                 : "memory");
}

struct MmaParams {
    SwitchParams base;
    const CUtensorMap* tmaps_ld;   // per segment: 32 x 64 swizzled box on the source (live or pristine)
    const CUtensorMap* tmaps_st;   // per segment: the same box shape on the live matrix
    int n_stages;                  // ring depth actually used (<= MmaLayout<KS>::stages)
    int store_depth;               // tile stores that may still be reading shared memory (0..3)
};

// Gated DOWN slab for one unit: rows [0, S) hold hi(g*a), rows [s_pad, s_pad+S) hold lo; the
// padding rows up to s_pad are zero.  Staging is split in two so the global-load latency hides
// under a whole unit of tiles: down_prefetch() issues this thread's 16-byte loads of the NEXT
// unit's DOWN rows into registers, down_commit() folds the gate (one f32 multiply,
// adapters.py:202), splits into bf16 hi + lo and writes the slab.
template <int KS>
__device__ __forceinline__ void down_prefetch(uint4 (&regs)[KS], const SegDev& sg, const Plan& plan, int S, int col0,
                                              int tid) {
    constexpr int chunks_per_row = kTN / 8;
    const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(sg.down);
    const int r = sg.rank;
#pragma unroll
    for (int j = 0; j < KS; ++j) {
        const int i = tid + j * kMmaConsumers;
        const int q = i / chunks_per_row;
        const int c = (i % chunks_per_row) * 8;
        regs[j] = make_uint4(0u, 0u, 0u, 0u);
        if (q < S && col0 + c < sg.d_in) {
            const int b = q / r, qr = q % r;
            regs[j] = __ldg(reinterpret_cast<const uint4*>(base + (long long)plan.expert[b] * sg.down_estride +
                                                           (long long)qr * sg.ld_down + col0 + c));
        }
    }
}

template <int KS>
__device__ __forceinline__ void down_commit(unsigned char* down_smem, const uint4 (&regs)[KS], int rank, const Plan& plan,
                                            int S, int tid) {
    constexpr int s_pad = KS * 16;
    constexpr int chunks_per_row = kTN / 8;
#pragma unroll
    for (int j = 0; j < KS; ++j) {
        const int i = tid + j * kMmaConsumers;
        const int q = i / chunks_per_row;
        const int c = (i % chunks_per_row) * 8;
        uint4 hi = make_uint4(0u, 0u, 0u, 0u), lo = hi;
        if (q < S) {
            const float w = plan.weight[q / rank];
            const uint32_t in[4] = {regs[j].x, regs[j].y, regs[j].z, regs[j].w};
            uint32_t oh[4], ol[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float f0 = __fmul_rn(w, bf16lo_to_f32(in[e]));
                const float f1 = __fmul_rn(w, bf16hi_to_f32(in[e]));
                const uint32_t h = pack_bf16x2(f0, f1);
                oh[e] = h;
                ol[e] = pack_bf16x2(f0 - bf16lo_to_f32(h), f1 - bf16hi_to_f32(h));
            }
            hi = make_uint4(oh[0], oh[1], oh[2], oh[3]);
            lo = make_uint4(ol[0], ol[1], ol[2], ol[3]);
        }
        *reinterpret_cast<uint4*>(down_smem + ((size_t)q * kDownPitch + c) * 2) = hi;
        *reinterpret_cast<uint4*>(down_smem + ((size_t)(s_pad + q) * kDownPitch + c) * 2) = lo;
    }
}

using MmaIter = TileIterT<kMR>;

// Warp roles (all walk the same static tile sequence):
//   warps 0..15  consumers: wait full[stage] -> W + U.(hi+lo) in place in smem -> arrive computed[stage]
//   W producers  (kWProd warps, 1 thread each): wait empty[stage] -> TMA loads of their W boxes
//   UP producer  (1 warp, 1 thread): wait empty[stage] -> bulk copies of the selected UP blocks
//   storers      (kStorers warps, 1 thread each): wait computed[stage] -> TMA stores of their
//                boxes; a stage goes back to the producers once every storer's stores have read
//                shared memory (store_depth newer stores may still be draining)
template <int KS>
__global__ void __launch_bounds__(kMmaThreads, 1) switch_mma_kernel(const __grid_constant__ MmaParams mp) {
    using L = MmaLayout<KS>;
    constexpr int kSt = L::stages < kMmaDefaultStages ? L::stages : kMmaDefaultStages;
    extern __shared__ unsigned char smem_dyn[];
    const SwitchParams& p = mp.base;
    // 128-byte swizzle needs 1024-byte aligned boxes
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::off_bar);
    uint64_t* computed = full + 16;
    uint64_t* empty = full + 32;
    Plan& plan = *reinterpret_cast<Plan*>(sm + L::off_plan);
    const int tid = threadIdx.x;

    if (tid == 0) {
        for (int s = 0; s < kSt; ++s) {
            mbar_init(&full[s], kWProd + 1);
            mbar_init(&computed[s], kMmaWarps);
            mbar_init(&empty[s], kStorers);
        }
        fence_mbar_init();
        if (p.use_dev)
            build_plan(plan, p.from_pristine ? nullptr : p.prev_dev, p.cur_dev, p.scale, false, p.n_experts_limit);
        else
            plan = p.host_plan;
        if (!plan_usable(p, plan, p.prev_dev, p.cur_dev)) plan.n_blocks = -1;
    }
    __syncthreads();
    const int n_blocks = plan.n_blocks;
    if (n_blocks < 0) return;                       // unusable decision: flagged, nothing touched
    if (n_blocks == 0 && !p.from_pristine) return;  // unchanged decision: nothing to move

    const uint32_t w_base = smem_u32(sm + L::off_w);
    const uint32_t up_base = smem_u32(sm + L::off_up);
    const int warp = tid >> 5, lane = tid & 31;

    // One thread can issue a TMA operation only every ~100 cycles; at 16 KB per stage a single
    // producer thread would be the bottleneck of the whole kernel (measured: 4.80 ms -> 4.29 ms on
    // the Llama-2-7B table when the UP copies moved to their own thread).  The issue work is
    // therefore spread over kWProd W-load threads, one UP-copy thread and kStorers store threads.
    if (warp >= kMmaWarps && warp < kMmaWarps + kWProd) {
        // ============ W producers: boxes b = who, who + kWProd, ... of every tile ============
        if (lane == 0) {
            const int who = warp - kMmaWarps;
            constexpr int kMine = (kBoxes + kWProd - 1) / kWProd;
            MmaIter ti;
            ti.init(p);
            for (int it = 0; ti.valid(p); ++it) {
                const int stage = it % kSt;
                const uint32_t ph = (it / kSt) & 1;
                mbar_wait(&empty[stage], ph ^ 1);
                int mine = 0;
#pragma unroll
                for (int j = 0; j < kMine; ++j) mine += (who + j * kWProd < kBoxes) ? 1 : 0;
                mbar_expect_tx(&full[stage], mine * kBoxBytes);
                const CUtensorMap* tm = mp.tmaps_ld + ti.un.seg;
#pragma unroll
                for (int j = 0; j < kMine; ++j) {
                    const int b = who + j * kWProd;
                    if (b < kBoxes)
                        tma_load_2d_addr(w_base + stage * kWStageBytes + b * kBoxBytes, tm, ti.un.col0 + b * kBoxCols, ti.m0,
                                         &full[stage]);
                }
                ti.next(p);
            }
        }
        return;
    }
    if (warp == kMmaWarps + kWProd) {
        // ============ UP producer: one 1-D bulk copy per selected expert block ============
        if (lane == 0) {
            MmaIter ti;
            ti.init(p);
            SegDev sg;
            int cur_seg = -1;
            for (int it = 0; ti.valid(p); ++it) {
                const int stage = it % kSt;
                const uint32_t ph = (it / kSt) & 1;
                if (ti.un.seg != cur_seg) {
                    cur_seg = ti.un.seg;
                    sg = p.segs[cur_seg];
                }
                const int rows_here = min(kMR, sg.d_out - ti.m0);
                const uint32_t up_blk_bytes = (uint32_t)rows_here * sg.rank * 2;
                mbar_wait(&empty[stage], ph ^ 1);
                mbar_expect_tx(&full[stage], n_blocks * up_blk_bytes);
                const __nv_bfloat16* upb = reinterpret_cast<const __nv_bfloat16*>(sg.up);
                for (int b = 0; b < n_blocks; ++b)
                    bulk_load_1d(up_base + stage * L::up_stage_bytes + b * (kMR * sg.rank * 2),
                                 upb + (long long)plan.expert[b] * sg.up_estride + (long long)ti.m0 * sg.rank,
                                 up_blk_bytes, &full[stage]);
                ti.next(p);
            }
        }
        return;
    }
    if (warp > kMmaWarps + kWProd) {
        // ============ storers: boxes back to global, then hand the stage back ============
        if (lane == 0) {
            const int who = warp - (kMmaWarps + kWProd + 1);
            constexpr int kMine = (kBoxes + kStorers - 1) / kStorers;
            MmaIter ti;
            ti.init(p);
            int it = 0;
            for (; ti.valid(p); ++it) {
                const int stage = it % kSt;
                const uint32_t ph = (it / kSt) & 1;
                mbar_wait(&computed[stage], ph);
                const CUtensorMap* tm = mp.tmaps_st + ti.un.seg;
#pragma unroll
                for (int j = 0; j < kMine; ++j) {
                    const int b = who + j * kStorers;
                    if (b < kBoxes)
                        tma_store_2d_addr(tm, ti.un.col0 + b * kBoxCols, ti.m0, w_base + stage * kWStageBytes + b * kBoxBytes);
                }
                bulk_commit();
                // the stores of tile it - depth have drained their stage: hand it back
                const int depth = mp.store_depth;
                if (depth <= 0) bulk_wait_read<0>();
                else if (depth == 1) bulk_wait_read<1>();
                else if (depth == 2) bulk_wait_read<2>();
                else bulk_wait_read<3>();
                if (it >= depth) mbar_arrive(&empty[(it - depth) % kSt]);
                ti.next(p);
            }
            bulk_wait_all<0>();  // global writes complete before the CTA retires
        }
        return;
    }

    // ================================ consumers ====================================
    const int mi = lane >> 3, rr = lane & 7;       // ldmatrix: lane supplies row rr of matrix mi
    const int wbox = warp >> 2;                    // this warp: 16 columns = chunks (warp & 3) * 2 + {0, 1} of box wbox
    const int wchunk = (warp & 3) * 2 + (mi >> 1);
    const int ncol = warp * 16 + (mi >> 1) * 8;    // slab column this lane addresses
    unsigned char* down_smem = sm + L::off_down;
    const uint32_t down_base = smem_u32(down_smem);

    MmaIter ti;
    ti.init(p);
    if (!ti.valid(p)) return;
    SegDev sg = p.segs[ti.un.seg];
    int S = n_blocks * sg.rank;
    uint4 dn_regs[KS];
    down_prefetch<KS>(dn_regs, sg, plan, S, ti.un.col0, tid);
    down_commit<KS>(down_smem, dn_regs, sg.rank, plan, S, tid);
    named_bar_sync(1, kMmaConsumers);  // first slab visible
    bool new_unit = true;
    uint32_t bfr[2][KS][4];
    SegDev sg_next = sg;
    int S_next = 0;
    bool have_next = false;
    for (int it = 0; ti.valid(p); ++it) {
        const int stage = it % kSt;
        const uint32_t ph = (it / kSt) & 1;
        if (new_unit) {
            // B fragments of this unit's slab -> registers (kept for every tile of the unit)
#pragma unroll
            for (int half = 0; half < 2; ++half)
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    const int krow = half * L::s_pad + 16 * j + (mi & 1) * 8 + rr;
                    ldmatrix_x4_trans(bfr[half][j], down_base + (krow * kDownPitch + ncol) * 2);
                }
            // start fetching the NEXT unit's DOWN rows; they are committed to the slab at its start
            const int un = ti.u + gridDim.x;
            have_next = un < p.n_units;
            if (have_next) {
                const UnitDev nu = p.units[un];
                sg_next = p.segs[nu.seg];
                S_next = n_blocks * sg_next.rank;
                down_prefetch<KS>(dn_regs, sg_next, plan, S_next, nu.col0, tid);
            }
        }
        new_unit = ti.next(p);

        mbar_wait(&full[stage], ph);
        const uint32_t w_stage = w_base + stage * kWStageBytes + wbox * kBoxBytes;
        const uint32_t up_stage = up_base + stage * L::up_stage_bytes;
#pragma unroll
        for (int mt = 0; mt < kMR / 16; ++mt) {
            const int row = mt * 16 + (mi & 1) * 8 + rr;  // tile row this lane addresses
            const uint32_t waddr = w_stage + row * 128 + ((wchunk ^ (row & 7)) << 4);
            uint32_t wv[4];
            ldmatrix_x4(wv, waddr);
            // A fragments (UP rows); ranks past S are padding and read as 0 (the slab rows are 0 too)
            uint32_t afrag[KS][4];
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const int k0 = 16 * j + (mi >> 1) * 8;  // first rank of the 8x8 matrix this lane addresses
                const int kk = k0 < S ? k0 : 0;
                const int b = kk / sg.rank, kin = kk % sg.rank;
                ldmatrix_x4(afrag[j], up_stage + ((b * kMR + row) * sg.rank + kin) * 2);
                if (16 * j >= S) afrag[j][0] = afrag[j][1] = 0u;
                if (16 * j + 8 >= S) afrag[j][2] = afrag[j][3] = 0u;
            }
            float acc[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
#pragma unroll
            for (int half = 0; half < 2; ++half)
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    mma_bf16_16816(acc[0], afrag[j], bfr[half][j][0], bfr[half][j][1]);
                    mma_bf16_16816(acc[1], afrag[j], bfr[half][j][2], bfr[half][j][3]);
                }
            // W + D, rounded RNE to bf16, written back in place (swizzled smem)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const uint32_t a = wv[nt * 2], b2 = wv[nt * 2 + 1];
                wv[nt * 2] = pack_bf16x2(bf16lo_to_f32(a) + acc[nt][0], bf16hi_to_f32(a) + acc[nt][1]);
                wv[nt * 2 + 1] = pack_bf16x2(bf16lo_to_f32(b2) + acc[nt][2], bf16hi_to_f32(b2) + acc[nt][3]);
            }
            stmatrix_x4(waddr, wv);
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the TMA store
        __syncwarp();
        if (lane == 0) mbar_arrive(&computed[stage]);

        if (new_unit && have_next) {
            named_bar_sync(1, kMmaConsumers);  // every warp holds its B fragments: the slab may be rewritten
            sg = sg_next;
            S = S_next;
            down_commit<KS>(down_smem, dn_regs, sg.rank, plan, S, tid);
            named_bar_sync(1, kMmaConsumers);  // next slab visible
        }
    }
}

}  // namespace af
