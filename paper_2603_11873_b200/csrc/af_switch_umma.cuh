// af_switch_umma.cuh -- the fused switch (+ GEMV) with the rank-s product on the 5th-generation
// tensor cores: tcgen05.mma issued by ONE thread, accumulators in tensor memory (TMEM).
//
// Why: the mma.sync tile loop of af_switch_mma.cuh is consumer-bound (profiles/README.md): 16 warps
// spend ~130 instructions per warp and 16 KB tile feeding the tensor pipe (ldmatrix of UP, B
// fragments in registers, 16 HMMA, fragment bookkeeping) -- 0.8 us per tile against 0.72 us of HBM
// time.  Here the product  D[128 x 128] = U[128 x 8 n_blocks] . (hi + lo)(g A)[8 n_blocks x 128]  is
// 2 * ceil(n_blocks / 2) tcgen05.mma instructions from one warp (an elected lane), straight from shared memory:
//   A = the UP ring as it is loaded -- one expert block (128 rows x 8 ranks) is a contiguous
//       [128][16 B] slab = one K-chunk of the K-major no-swizzle canonical layout (LBO = slab
//       stride, SBO = 128 B);
//   B = the gated DOWN slab written in the MN-major no-swizzle canonical layout (8 k x 8 n core
//       matrices; n-groups 128 B apart, k-groups = blocks 2 KB apart), hi blocks then lo blocks;
//   D = f32 in TMEM, two 128-column accumulators so the MMAs of tile t+1 run under the epilogue of t.
// The epilogue warps own one row each (TMEM lane = row): tcgen05.ld 32 columns, add the W row
// from the swizzled TMA tile, round to bf16, store back, and -- fused GEMV -- dot the rounded row
// with the staged input strip; the row's partial sum goes straight to the fixed-point accumulator
// (no cross-warp reduction: a thread holds the whole 128-column row strip).
//
// Scope: tables of ONE rank in {8, 16, 32, 64}, matrices multiples of 128 in both directions (every
// Llama shape of BASELINE.json).  Stacked ranks: up to 256 in ONE launch (K-chunked, below) for ranks 8 / 16 /
// 32; rank 64 up to 64.  (scripts/micro/umma_test.cu pins the descriptor encodings in isolation.)
//
// K-chunking (template argument CH < NB): the reference's merge is ONE sgmm whatever the stacked rank
// (adapters.py:236-258 -> linalg.py:306-346).  With more than 32 stacked ranks the UP operand of a tile no
// longer fits the ring next to the W tiles, so it streams through the UP ring in CHUNKS of 32 ranks (8 KB:
// CH = 4 k-groups of 8) while the tile's accumulator stays in tensor memory: per chunk 2 x 2 tcgen05.mma
// (hi and lo halves of the resident slab, K = 16 each), a commit that frees the chunk's stage, and after
// the last chunk the commit that hands the accumulator to the epilogue.  One read and one write of W and
// ONE bf16 rounding per token at any stacked rank up to 256 (Llama-2-70B, r = 32, k = 4) -- the multi-pass
// schedule this replaces read and rounded W once per 64 ranks.
#pragma once

#include "af_switch_mma.cuh"

namespace af {

constexpr int kUM = 128;                           // tile rows  (UMMA M)
constexpr int kUN = 128;                           // tile cols  (UMMA N) = strip width
constexpr int kUBoxCols = 64;                      // TMA box: 128 rows x 64 cols, 128-byte swizzle
constexpr int kUBoxes = kUN / kUBoxCols;           // 2
constexpr int kUBoxBytes = kUM * kUBoxCols * 2;    // 16 KB
constexpr int kUWStage = kUM * kUN * 2;            // 32 KB
constexpr int kUBlockBytes = kUM * 8 * 2;          // one expert block of the UP stage: 128 rows x 8 ranks = 2 KB
constexpr int kUSlabBlock = 8 * kUN * 2;           // one k-group (8 ranks) of the slab: 2 KB
constexpr int kUEpiWarps = 8;                      // two groups of 4: TMEM lane quarter = warp % 4
constexpr int kUEpi = kUEpiWarps * 32;
constexpr int kUThreads = kUEpi + 4 * 32;          // + W producer, UP producer, MMA issuer, storer
constexpr int kUXSlots = 4;
#ifndef AF_UMMA_PF
#define AF_UMMA_PF 0   /* measured: prefetching W into L2 beyond the ring costs 20 % (profiles/README.md) */
#endif
constexpr int kUPrefetch = AF_UMMA_PF;             // W tiles prefetched into L2 beyond the shared-memory ring (0 = off)
#ifndef AF_UMMA_BURST
#define AF_UMMA_BURST 4
#endif
#ifndef AF_UMMA_BURST_AFTER
#define AF_UMMA_BURST_AFTER 5000   /* cycles (~2.5 us) the ring must have stayed full before the loader prefetches ahead */
#endif
constexpr int kUBurst = AF_UMMA_BURST;             // tiles pulled into L2 when the consumers stall (phase boundary)
constexpr long long kUBurstAfterCycles = AF_UMMA_BURST_AFTER;

// NB = k-groups of 8 stacked ranks the slab holds per half; CH = k-groups per UP ring stage (CH == NB: the whole
// UP operand of a tile is one stage; CH < NB: K-chunked, NB / CH chunks per tile)
// PC = bf16 pieces the gated DOWN rows are split into: 2 (hi + lo: g*a reproduced to 2^-17) or 3 (hi + mid + lo: the f32 value
// of g*a exactly -- 24 bits in three 8-bit pieces -- so that the product differs from the reference's f32 merge only by the
// order of the f32 sums).  Three pieces need 50 % more slab and MMAs: offered where both are cheap, at up to 32 stacked ranks
// (af_set_umma_pieces(3): 8x fewer last-bit differences against the oracle for 0.4 % of the Llama-2-7B step at full clocks,
// 1.5 % on a power-capped board; the default stays two -- the mma.sync kernels' split, so both tensor paths agree to the bit
// count the tests pin).
template <int NB, bool GEMV, int CH = NB, int PC = 2>
struct UmmaLayout {
    static_assert(NB % CH == 0 && CH % 2 == 0, "chunks are whole rank-16 steps");
    static_assert(PC == 2 || (PC == 3 && NB <= 4 && CH == NB), "three pieces: launches of at most 32 stacked ranks");
    static constexpr bool chunked = CH < NB;
    static constexpr int up_stage = CH * kUBlockBytes;
    static constexpr int slab_bytes = PC * NB * kUSlabBlock;           // hi + lo (+ a third piece)
    static constexpr int xs_bytes = GEMV ? kUXSlots * kUN * 4 : 0;
    static constexpr int misc = 1024 /*barriers*/ + (int)sizeof(Plan) + 256 + kUnitCache * (int)sizeof(UnitDev) + kSegCache * (int)sizeof(SegDev);
    static constexpr int fixed = slab_bytes + xs_bytes + misc + 2048;
    // Two rings.  W tiles (32 KB, from HBM) live from their load until their store has read them; UP stages
    // (from L2) only until the MMAs that read them have completed, two tiles ahead of the epilogue at most.
    // Whole-operand stages: three are enough, which leaves a 64-rank launch (16 KB UP stages, 32 KB slab) four
    // W stages instead of three.  Chunked: a tile consumes NB / CH stages in a burst, each an L2 round trip.  With
    // 32-rank chunks (8 KB): six stages (measured at 128 stacked ranks on Llama-2-70B shard shapes: six UP + three W
    // stages 2.59 ms, three UP + four W stages 2.85 ms) -- except at 256, where the 128 KB slab leaves room for three
    // UP and two W stages.  With 64-rank chunks (16 KB, the choice at 128 stacked ranks: 2.41 ms): three stages.
    static constexpr int up_stages_wanted = chunked ? ((NB >= 32 || CH >= 8) ? 3 : 6) : (NB > 4 ? 3 : 6);
    static constexpr int by_smem = (227 * 1024 - fixed) / (kUWStage + up_stage);          // equal depths
    static constexpr int by_smem_w = (227 * 1024 - fixed - up_stages_wanted * up_stage) / kUWStage;
    // (three pieces at 32 stacked ranks: the 24 KB slab would cost a W stage at equal depths; four UP stages keep five W stages)
    static constexpr int stages = PC == 3 ? 5 : (NB > 4 || chunked) ? (by_smem_w < 6 ? by_smem_w : 6) : (by_smem < 6 ? by_smem : 6);
    static constexpr int up_stages = PC == 3 ? 4 : (NB > 4 || chunked) ? up_stages_wanted : stages;
    static constexpr int off_w = 0;
    static constexpr int off_up = off_w + stages * kUWStage;
    static constexpr int off_slab = off_up + up_stages * up_stage;     // 1024-aligned (multiples of 2 KB)
    static constexpr int off_xs = off_slab + slab_bytes;
    static constexpr int off_bar = off_xs + xs_bytes;
    static constexpr int off_plan = off_bar + 1024;
    static constexpr int off_red = (off_plan + (int)sizeof(Plan) + 15) & ~15;
    static constexpr int off_units = off_red + 256;
    static constexpr int off_segs = off_units + kUnitCache * (int)sizeof(UnitDev);
    static constexpr int total = off_segs + kSegCache * (int)sizeof(SegDev) + 1024;
    static_assert(stages >= 2 && up_stages >= 3 && up_stages <= 8 && total <= 227 * 1024, "shared memory budget");
};

// ---- tcgen05 wrappers ----
// layout: 0 = no swizzle, 6 / 4 / 2 = 32- / 64- / 128-byte swizzle (UMMA::LayoutType)
__device__ __forceinline__ uint64_t umma_desc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout = 0) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version of sm_100
    d |= (uint64_t)(layout & 7) << 61;
    return d;
}
// A operand (UP stage) of the rank-16 step ks.  rank 8: an expert block is a [128][16 B] slab, two blocks make a
// step (no swizzle, LBO = block stride).  rank 16 / 32 / 64: the block came through a tensor map whose swizzle
// span is the row (32 / 64 / 128 bytes), which IS the K-major swizzled canonical layout; a step is 32 bytes
// further along the row, blocks follow each other.
__device__ __forceinline__ uint64_t umma_a_desc(uint32_t up_stage, int rank, int ks) {
    if (rank == 8) return umma_desc(up_stage + ks * 2 * kUBlockBytes, kUBlockBytes, 128);
    const int k0 = 16 * ks, b = k0 / rank, ko = k0 % rank;
    const uint32_t layout = rank == 16 ? 6u : (rank == 32 ? 4u : 2u);
    return umma_desc(up_stage + b * (kUM * rank * 2) + ko * 2, 16, 8 * rank * 2, layout);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}
// The same, for a converged warp: every lane executes it, elect.sync picks the one that issues.
__device__ __forceinline__ void umma_bf16_elect(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|q, 0xffffffff;\n\t"
        "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\t"
        "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// TMA prefetch of one box into L2 (no shared memory, no barrier)
__device__ __forceinline__ void tma_prefetch_l2_2d(const void* tmap, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tmap), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,"
        "%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
          "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// tile walk with 128-row tiles (units are cut at multiples of kUM)
// This CTA's partial sums of phases [from, to) are out: bump their counters (after the fence that orders the atomics
// before the bump).  A phase that was pushed to the peers (MmaParams::reduce_mask) is reported on every rank's counter.
template <bool PEERS>
__device__ __forceinline__ void umma_publish_phases(const MmaParams& mp, int from, int to) {
    if (from >= to) return;
    if (PEERS && mp.n_peers > 0) __threadfence_system();
    else __threadfence();
    for (int ph = from; ph < to; ++ph) {
        if (PEERS && mp.n_peers > 0 && ((mp.reduce_mask >> ph) & 1)) {
            for (int w = 0; w < mp.n_peers; ++w)
                atomicAdd_system(reinterpret_cast<int*>(reinterpret_cast<char*>(mp.phase_done + ph) + mp.peer_off[w]), 1);
        } else {
            atomicAdd(mp.phase_done + ph, 1);
        }
    }
}
// Counters a launch bumps: one per phase boundary, plus the last phase's when that one is reduced over the peers
// (its consumer is a later launch, which waits for it with af_peer_wait).
template <bool PEERS>
__device__ __forceinline__ int umma_phases_to_publish(const MmaParams& mp) {
    const bool last_reduced = PEERS && mp.n_peers > 0 && ((mp.reduce_mask >> (mp.n_phases - 1)) & 1);
    return mp.n_phases - 1 + (last_reduced ? 1 : 0);
}

struct UmmaIter {
    int j, u, m0, row_end;
    UnitDev un;
    const UnitDev* cache;
    __device__ __forceinline__ bool valid(const SwitchParams& p) const { return u < p.n_units; }
    __device__ __forceinline__ UnitDev fetch(const SwitchParams& p, int jj, int uu) const { return jj < kUnitCache ? cache[jj] : p.units[uu]; }
    __device__ __forceinline__ void load_unit(const SwitchParams& p) {
        if (u < p.n_units) {
            un = fetch(p, j, u);
            m0 = un.row0;
            row_end = un.row0 + un.rows;
            if (un.rows <= 0) u = p.n_units;
        }
    }
    __device__ __forceinline__ void init(const SwitchParams& p, const UnitDev* c) {
        cache = c;
        j = 0;
        u = blockIdx.x;
        load_unit(p);
    }
    __device__ __forceinline__ bool next(const SwitchParams& p) {
        m0 += kUM;
        if (m0 < row_end) return false;
        u += gridDim.x;
        ++j;
        load_unit(p);
        return true;
    }
    __device__ __forceinline__ UnitDev peek(const SwitchParams& p) const {
        const int un2 = u + gridDim.x;
        if (un2 >= p.n_units) return UnitDev{0, 0, 0, 0, 0, 0};
        return fetch(p, j + 1, un2);
    }
};

// Gated DOWN slab of one unit in the MN-major canonical layout: element (rank row q, column n) at
//   (q / 8) * 2 KB + (n / 8) * 128 B + (q % 8) * 16 B + (n % 8) * 2 B ;  lo blocks NB k-groups after the hi blocks.
// Staged in two steps like the mma.sync kernel's: umma_slab_prefetch() issues this thread's 16-byte
// loads of the NEXT unit's DOWN rows (predicated asm: nothing consumes them yet, so nothing waits),
// umma_slab_commit() folds the gate, splits into bf16 hi + lo and writes the slab.
template <int NB>
__device__ __forceinline__ void umma_slab_prefetch(uint4 (&regs)[NB * 8 * (kUN / 8) / kUEpi], const SegDev& sg, const Plan& plan, int S,
                                                   int col0, int tid) {
    constexpr int chunks = kUN / 8;                 // 16-byte chunks per rank row
    const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(sg.down);
#pragma unroll
    for (int j = 0; j < NB * 8 * chunks / kUEpi; ++j) {
        const int i = tid + j * kUEpi;
        const int q = i / chunks, c = (i % chunks) * 8;
        const bool ok = q < S && col0 + c < sg.d_in;
        const int qq = ok ? q : 0;
        int qb, qr;
        rank_divmod(qq, sg.rank, qb, qr);
        const __nv_bfloat16* src = base + (long long)plan.expert[qb] * sg.down_estride + (long long)qr * sg.ld_down + col0 + c;
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %5, 0;\n"
            "mov.b32 %0, 0;\n"
            "mov.b32 %1, 0;\n"
            "mov.b32 %2, 0;\n"
            "mov.b32 %3, 0;\n"
            "@p ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];\n"
            "}\n"
            : "=r"(regs[j].x), "=r"(regs[j].y), "=r"(regs[j].z), "=r"(regs[j].w)
            : "l"(ok ? src : base), "r"((int)ok));
    }
}
template <int NB, int PC>
__device__ __forceinline__ void umma_slab_commit(unsigned char* slab, const uint4 (&regs)[NB * 8 * (kUN / 8) / kUEpi], const Plan& plan, int S,
                                                 int rank, int tid) {
    constexpr int chunks = kUN / 8;
#pragma unroll
    for (int j = 0; j < NB * 8 * chunks / kUEpi; ++j) {
        const int i = tid + j * kUEpi;
        const int q = i / chunks, c = (i % chunks) * 8;
        uint4 hi = make_uint4(0u, 0u, 0u, 0u), lo = hi, lo2 = hi;
        if (q < S) {
            int wb, wr;
            rank_divmod(q, rank, wb, wr);
            const float w = plan.weight[wb];
            const uint32_t in[4] = {regs[j].x, regs[j].y, regs[j].z, regs[j].w};
            uint32_t oh[4], ol[4], ol2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float f0 = __fmul_rn(w, bf16lo_to_f32(in[e]));       // one rounding, as the reference folds the gate (adapters.py:202)
                const float f1 = __fmul_rn(w, bf16hi_to_f32(in[e]));
                const uint32_t h = pack_bf16x2(f0, f1);
                oh[e] = h;
                const float r0 = f0 - bf16lo_to_f32(h), r1 = f1 - bf16hi_to_f32(h);   // exact in f32
                const uint32_t m = pack_bf16x2(r0, r1);
                ol[e] = m;
                if constexpr (PC == 3) ol2[e] = pack_bf16x2(r0 - bf16lo_to_f32(m), r1 - bf16hi_to_f32(m));   // exact: 24 bits = 8 + 8 + 8
            }
            hi = make_uint4(oh[0], oh[1], oh[2], oh[3]);
            lo = make_uint4(ol[0], ol[1], ol[2], ol[3]);
            if constexpr (PC == 3) lo2 = make_uint4(ol2[0], ol2[1], ol2[2], ol2[3]);
        }
        const int off = (q >> 3) * kUSlabBlock + (c >> 3) * 128 + (q & 7) * 16;
        *reinterpret_cast<uint4*>(slab + off) = hi;
        *reinterpret_cast<uint4*>(slab + NB * kUSlabBlock + off) = lo;
        if constexpr (PC == 3) *reinterpret_cast<uint4*>(slab + 2 * NB * kUSlabBlock + off) = lo2;
    }
}

// The same staging without the register hand-over, for slabs too large to park in registers across a unit
// (NB > 8: 16 and more 16-byte words per thread): loaded and committed four words at a time at the unit's start.
template <int NB>
__device__ __forceinline__ void umma_slab_direct(unsigned char* slab, const SegDev& sg, const Plan& plan, int S, int col0, int tid) {
    constexpr int chunks = kUN / 8;
    constexpr int per_thread = NB * 8 * chunks / kUEpi;
    static_assert(per_thread % 4 == 0, "four words in flight");
    const __nv_bfloat16* base = reinterpret_cast<const __nv_bfloat16*>(sg.down);
#pragma unroll 1
    for (int j0 = 0; j0 < per_thread; j0 += 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = tid + (j0 + u) * kUEpi;
            const int q = i / chunks, c = (i % chunks) * 8;
            v[u] = make_uint4(0u, 0u, 0u, 0u);
            if (q < S && col0 + c < sg.d_in) {
                int qb, qr;
                rank_divmod(q, sg.rank, qb, qr);
                v[u] = __ldg(reinterpret_cast<const uint4*>(base + (long long)plan.expert[qb] * sg.down_estride + (long long)qr * sg.ld_down + col0 + c));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = tid + (j0 + u) * kUEpi;
            const int q = i / chunks, c = (i % chunks) * 8;
            uint4 hi = make_uint4(0u, 0u, 0u, 0u), lo = hi;
            if (q < S) {
                int wb, wr;
                rank_divmod(q, sg.rank, wb, wr);
                const float w = plan.weight[wb];
                const uint32_t in[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
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
            const int off = (q >> 3) * kUSlabBlock + (c >> 3) * 128 + (q & 7) * 16;
            *reinterpret_cast<uint4*>(slab + off) = hi;
            *reinterpret_cast<uint4*>(slab + NB * kUSlabBlock + off) = lo;
        }
    }
}

// PEERS: the tensor-parallel pushes (MmaParams::n_peers) are compiled in -- a separate instantiation, so that a single
// rank's kernel carries none of it (measured: 0.4 % of the Llama-2-7B step otherwise)
template <int NB, bool GEMV, int CH = NB, int PC = 2, bool PEERS = false>
__global__ void __launch_bounds__(kUThreads, 1) switch_umma_kernel(const __grid_constant__ MmaParams mp) {
    using L = UmmaLayout<NB, GEMV, CH, PC>;
    constexpr bool kPrefetchSlab = NB <= 8;   // the next unit's DOWN rows wait in registers (umma_slab_prefetch)
    constexpr int kSt = L::stages, kUpSt = L::up_stages;
    extern __shared__ unsigned char smem_dyn[];
    const SwitchParams& p = mp.base;
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::off_bar);   // [8]
    uint64_t* computed = full + 8;                                    // [8]
    uint64_t* empty = full + 16;                                      // [8]
    uint64_t* acc_full = full + 24;                                   // [2]
    uint64_t* acc_empty = full + 26;                                  // [2]
    uint64_t* slab_bar = full + 28;                                   // [1]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(full + 30);
    uint64_t* up_full = full + 32;                                    // [8]  UP ring: loaded by the UP producer ...
    uint64_t* up_empty = full + 40;                                   // [8]  ... released when the tile's MMAs have completed
    Plan& plan = *reinterpret_cast<Plan*>(sm + L::off_plan);
    UnitDev* unit_cache = reinterpret_cast<UnitDev*>(sm + L::off_units);
    SegDev* seg_cache = reinterpret_cast<SegDev*>(sm + L::off_segs);
    // (the warp index through a shuffle: the compiler then knows the role branches are warp-uniform)
    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;

    unsigned long long* const tl = GEMV ? mp.timeline : nullptr;   // probe: a few stamps per phase, none per tile
    if (tid == 0) tl_stamp(tl, 0);
    if (tid >= 32 && tid < 32 + kUnitCache) {
        const int jj = tid - 32;
        const long long uu = (long long)blockIdx.x + (long long)jj * gridDim.x;
        unit_cache[jj] = uu < p.n_units ? p.units[uu] : UnitDev{0, 0, 0, 0, 0, 0};
    }
    if (tid >= 64 && tid < 64 + mp.n_chain_segs) seg_cache[tid - 64] = p.segs[mp.chain_segs[tid - 64]];
    for (int i = tid * 16; i < kUpSt * L::up_stage; i += kUThreads * 16)   // block slots past n_blocks must read as zeros
        *reinterpret_cast<uint4*>(sm + L::off_up + i) = make_uint4(0u, 0u, 0u, 0u);
    if (tid == 0) {
        for (int s = 0; s < kSt; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&computed[s], 4);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < kUpSt; ++s) {
            mbar_init(&up_full[s], 1);
            mbar_init(&up_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        mbar_init(slab_bar, kUEpiWarps);
        *reinterpret_cast<volatile int*>(full + 31) = 0;
        fence_mbar_init();
        if (!p.plan_dev) {
            if (p.use_dev)
                build_plan(plan, p.from_pristine ? nullptr : p.prev_dev, p.cur_dev, p.scale, false, p.n_experts_limit);
            else
                plan = p.host_plan;
            if (!plan_usable(p, plan, p.prev_dev, p.cur_dev)) plan.n_blocks = -1;
        }
    }
    if (p.plan_dev) {
        constexpr int kWords = (int)(sizeof(Plan) / 4);
        if (tid >= 128 && tid < 128 + kWords) reinterpret_cast<int*>(&plan)[tid - 128] = reinterpret_cast<const int*>(p.plan_dev)[tid - 128];
    }
    if (warp == kUEpiWarps + 2) {   // the MMA warp owns the tensor memory: two 128-column accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_proxy_async_smem();       // zero-filled UP ring -> visible to the tensor core
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // (block-wide values read from shared memory, broadcast with a shuffle: the compiler cannot see that a load is
    //  warp-uniform, and only code under provably uniform branches gets the uniform datapath -- see the MMA issuer)
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    const int n_blocks = __shfl_sync(0xffffffffu, plan.n_blocks, 0);
    const bool store_w = n_blocks > 0 || p.from_pristine;
    const bool bail = n_blocks < 0 || (!GEMV && !store_w);
    const uint32_t w_base = smem_u32(sm + L::off_w), up_base = smem_u32(sm + L::off_up), slab_base = smem_u32(sm + L::off_slab);
    // chains cache their few segment descriptors in shared memory; a whole-table launch reads them from global
    auto seg_of = [&](const UnitDev& un) -> SegDev { return mp.n_chain_segs > 0 ? seg_cache[un.slot] : p.segs[un.seg]; };

    if (!bail) {
        if (warp == kUEpiWarps) {
            // ============ W producer: two 128 x 64 swizzled boxes per tile ============
            // Lane 1 runs ahead of it and prefetches the next kUPrefetch tiles into L2.  The ring alone holds
            // ~3 us of HBM time; a phase boundary stalls the consumers for ~5 us, during which the ring fills
            // up and HBM would go idle.  With the prefetcher the reads keep streaming (into L2), and after the
            // boundary the epilogue -- 4x faster than HBM -- catches up on tiles that now come from L2.
            if (lane == 1 && kUPrefetch > 0) {
                volatile int* prod_it = reinterpret_cast<volatile int*>(full + 31);
                UmmaIter ti;
                ti.init(p, unit_cache);
                for (int it = 0; ti.valid(p); ++it) {
                    while (it >= *prod_it + kUPrefetch) __nanosleep(64);   // at most kUPrefetch tiles beyond the loader
                    if (it >= kSt) {   // the first ring fill is loaded directly
                        const CUtensorMap* tm = mp.tmaps_ld + ti.un.seg;
#pragma unroll
                        for (int b = 0; b < kUBoxes; ++b) tma_prefetch_l2_2d(tm, ti.un.col0 + b * kUBoxCols, ti.m0);
                    }
                    ti.next(p);
                }
            }
            if (lane == 0) {
                const uint64_t pol = l2_evict_first_policy();
                UmmaIter ti;
                ti.init(p, unit_cache);
                // Stall burst (EXPERIMENT, off: AF_DBG=256 turns it on): when the ring has stayed full for longer than a
                // tile's worth of back-pressure the consumers sit at a phase boundary, and HBM idles until they are back
                // and the first stage comes free; the loader then pulls the next kUBurst tiles into L2 (TMA prefetch), so
                // that the ring would refill from L2 afterwards.  Measured on Llama-2-7B (round 2, A/B on one box, twice):
                // 5.58 against 5.52 ms per token WITHOUT it -- like the standing prefetcher of round 1 (-20 %), pulling W
                // into L2 ahead of the ring does not pay on this part; the boundary cost is not recoverable this way.
                UmmaIter tp = ti;
                int pf_it = 0;
                const bool burst_on = GEMV && kUBurst > 0 && (mp.dbg & 256);
                for (int it = 0; ti.valid(p); ++it) {
                    const int stage = it % kSt;
                    const uint32_t ph = (it / kSt) & 1;
                    *reinterpret_cast<volatile int*>(full + 31) = it + kSt;   // tiles up to it + kSt are the ring's business
                    if (burst_on && !mbar_test(&empty[stage], ph ^ 1)) {
                        const long long t0 = clock64();
                        bool fired = false;
                        while (!mbar_test(&empty[stage], ph ^ 1)) {
                            if (!fired && clock64() - t0 > kUBurstAfterCycles) {
                                fired = true;
                                if (pf_it < it) {   // the cursor never falls behind the loader
                                    pf_it = it;
                                    tp = ti;
                                }
                                while (pf_it < it + kUBurst && tp.valid(p)) {
                                    const CUtensorMap* tmp_ = mp.tmaps_ld + tp.un.seg;
#pragma unroll
                                    for (int b = 0; b < kUBoxes; ++b) tma_prefetch_l2_2d(tmp_, tp.un.col0 + b * kUBoxCols, tp.m0);
                                    tp.next(p);
                                    ++pf_it;
                                }
                            }
                        }
                    }
                    mbar_wait(&empty[stage], ph ^ 1);
                    mbar_expect_tx(&full[stage], kUWStage);
                    const CUtensorMap* tm = mp.tmaps_ld + ti.un.seg;
#pragma unroll
                    for (int b = 0; b < kUBoxes; ++b)
                        tma_load_2d_hint(w_base + stage * kUWStage + b * kUBoxBytes, tm, ti.un.col0 + b * kUBoxCols, ti.m0, &full[stage], pol);
                    ti.next(p);
                }
            }
        } else if (warp == kUEpiWarps + 1) {
            // ============ UP producer: one 2 KB bulk copy per selected expert block (rank 8), one swizzled box per
            // block otherwise; a tile's blocks go to one stage, or -- K-chunked -- to one stage per CH k-groups ============
            if (lane == 0) {
                UmmaIter ti;
                ti.init(p, unit_cache);
                SegDev sg;
                int cur_seg = -1;
                int uit = 0;
                for (int it = 0; ti.valid(p); ++it) {
                    if (ti.un.seg != cur_seg) {
                        cur_seg = ti.un.seg;
                        sg = seg_of(ti.un);
                    }
                    const uint32_t blk_bytes = (uint32_t)kUM * sg.rank * 2;
                    const int per_chunk = (CH * 8) / sg.rank;                      // expert blocks per stage
                    const int n_ch = n_blocks > 0 ? (n_blocks + per_chunk - 1) / per_chunk : 1;
                    for (int c = 0; c < n_ch; ++c, ++uit) {
                        const int stage = uit % kUpSt;
                        const uint32_t ph = (uit / kUpSt) & 1;
                        const int b0 = c * per_chunk, b1 = min(n_blocks, b0 + per_chunk);
                        mbar_wait(&up_empty[stage], ph ^ 1);
                        if (mp.dbg & 64) {   // timing experiment: no UP traffic at all
                            mbar_expect_tx(&up_full[stage], 0);
                            continue;
                        }
                        if (sg.rank == 8) {   // an expert block is 128 contiguous 16-byte rows: one bulk copy
                            // (a partial last row tile is cut at d_out: the rows behind it belong to the next expert, or to nobody;
                            //  what stays in the stage for them is finite and feeds accumulator rows that are never stored)
                            const uint32_t bytes = (uint32_t)min(kUM, sg.d_out - ti.m0) * 16u;
                            mbar_expect_tx(&up_full[stage], (uint32_t)max(0, b1 - b0) * bytes);
                            const __nv_bfloat16* upb = reinterpret_cast<const __nv_bfloat16*>(sg.up);
                            for (int b = b0; b < b1; ++b)
                                bulk_load_1d(up_base + stage * L::up_stage + (b - b0) * kUBlockBytes,
                                             upb + (long long)plan.expert[b] * sg.up_estride + (long long)ti.m0 * 8, bytes, &up_full[stage]);
                        } else {              // 128 rows x rank through the tensor map whose swizzle span is the row
                            mbar_expect_tx(&up_full[stage], (uint32_t)max(0, b1 - b0) * blk_bytes);
                            const CUtensorMap* tm = mp.tmaps_up + ti.un.seg;
                            for (int b = b0; b < b1; ++b)
                                tma_load_2d_addr(up_base + stage * L::up_stage + (b - b0) * blk_bytes, tm, 0, plan.expert[b] * sg.d_out + ti.m0,
                                                 &up_full[stage]);
                        }
                    }
                    ti.next(p);
                }
            }
        } else if (warp == kUEpiWarps + 2) {
            // ============ MMA issuer: D[buf] = U . hi + U . lo ============
            // The WHOLE warp runs this loop and elect.sync picks the lane that issues (umma_bf16_elect): with the warp
            // provably converged and every descriptor input warp-uniform (loop counters, shared-memory bases, values
            // broadcast with a shuffle), the compiler keeps the descriptors in uniform registers and an MMA costs the
            // issuing warp UIADD3 + UTCHMMA.  Under `if (lane == 0)` the same code compiled to an election loop with
            // five R2UR per MMA: 135 cycles of issue against the tensor core's 65 for M128 N128 K16
            // (scripts/micro/umma_rate.cu) -- the MMA stream, not HBM, was what bounded launches of 64+ stacked ranks.
            {
                // D f32, A / B bf16, A K-major, B MN-major, N = 128, M = 128
                constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(kUN >> 3) << 17) | ((uint32_t)(kUM >> 4) << 24);
                // The walk over this CTA's units (UmmaIter's order) with every branch condition warp-uniform: per unit
                // only its number of row tiles is needed, read by all lanes and broadcast.
                auto unit_tiles = [&](int jj, int uu) -> int {
                    int nt = 0;
                    if (uu < p.n_units) {
                        const int rows = jj < kUnitCache ? unit_cache[jj].rows : p.units[uu].rows;
                        nt = rows > 0 ? (rows + kUM - 1) / kUM : 0;
                    }
                    return __shfl_sync(0xffffffffu, nt, 0);
                };
                int unit_j = 0, unit_u = blockIdx.x;
                int nt = unit_tiles(unit_j, unit_u);
                int rank = 8;                                            // one rank for the whole table (eligibility)
                if (nt > 0) {
                    const UnitDev un0 = unit_cache[0];
                    rank = seg_of(un0).rank;
                }
                rank = __shfl_sync(0xffffffffu, rank, 0);
                const int nb_u = n_blocks;
                const uint32_t tmem_u = tmem;
                const int ksteps = (nb_u * rank + 15) >> 4;              // rank-16 steps over the stacked ranks
                const int per_chunk = (CH * 8) / rank;
                const int n_ch = nb_u > 0 ? (nb_u + per_chunk - 1) / per_chunk : 1;
                // the descriptors are a per-table prototype plus a precomputed 16-byte-unit offset per rank-16 step
                // (computing them from scratch -- divisions by the run-time rank -- cost ~2x the MMA itself)
                constexpr int kStepsPerChunk = CH / 2;
                uint32_t a_inc[kStepsPerChunk];
#pragma unroll
                for (int k2 = 0; k2 < kStepsPerChunk; ++k2)
                    a_inc[k2] = (uint32_t)(umma_a_desc(0u, rank, k2) & 0x3fffu);          // (offset inside a stage) >> 4
                const uint64_t a_proto = umma_a_desc(0u, rank, 0);                           // layout / LBO / SBO of the table's rank
                const uint64_t b_proto = umma_desc(0u, kUSlabBlock, 128);
                const uint32_t slab16 = slab_base >> 4;
                const int n_half = (mp.dbg & 32) ? 1 : PC;   // (dbg 32: timing experiment without the lo pieces)
                int it = 0, uit = 0;
                while (nt > 0) {
                    mbar_wait(slab_bar, (uint32_t)unit_j & 1);   // the unit's slab has been written (and made visible to the tensor core)
                    for (int t = 0; t < nt; ++t, ++it) {
                        const int buf = it & 1;
                        const uint32_t aph = (it >> 1) & 1;
                        mbar_wait(&acc_empty[buf], aph ^ 1);
                        const uint32_t d_tmem = tmem_u + buf * kUN;
                        uint32_t accumulate = 0;
                        for (int c = 0; c < n_ch; ++c, ++uit) {
                            const int stage = uit % kUpSt;
                            const uint32_t ph = (uit / kUpSt) & 1;
                            mbar_wait(&up_full[stage], ph);
                            tc_fence_after();
                            const uint32_t a16 = (up_base + stage * L::up_stage) >> 4;
                            const int ks0 = c * kStepsPerChunk;
                            for (int half = 0; half < n_half; ++half) {
                                const uint32_t b16 = slab16 + (uint32_t)((half * NB + ks0 * 2) * (kUSlabBlock >> 4));
#pragma unroll
                                for (int k2 = 0; k2 < kStepsPerChunk; ++k2) {
                                    if (ks0 + k2 < ksteps) {
                                        umma_bf16_elect(d_tmem, a_proto + (a16 + a_inc[k2]), b_proto + (b16 + (uint32_t)(k2 * 2 * (kUSlabBlock >> 4))),
                                                        idesc, accumulate);
                                        accumulate = 1;
                                    }
                                }
                            }
                            if (ksteps == 0)   // nothing selected (plain GEMV): D = 0 through a K = 16 product with the zeroed slot
                                umma_bf16_elect(d_tmem, a_proto + a16, b_proto + slab16, idesc, 0);
                            umma_commit_elect(smem_u32(&up_empty[stage]));   // the UP stage is free once these MMAs have read it
                        }
                        umma_commit_elect(smem_u32(&acc_full[buf]));          // every MMA of the tile has completed: the epilogue may read D
                    }
                    unit_u += gridDim.x;
                    ++unit_j;
                    nt = unit_tiles(unit_j, unit_u);
                }
            }
        } else if (warp == kUEpiWarps + 3) {
            // ============ storer ============
            if (lane == 0) {
                const uint64_t pol = l2_evict_first_policy();
                UmmaIter ti;
                ti.init(p, unit_cache);
                for (int it = 0; ti.valid(p); ++it) {
                    const int stage = it % kSt;
                    const uint32_t ph = (it / kSt) & 1;
                    mbar_wait(&computed[stage], ph);
                    if (store_w) {
                        const CUtensorMap* tm = mp.tmaps_st + ti.un.seg;
#pragma unroll
                        for (int b = 0; b < kUBoxes; ++b)
                            tma_store_2d_hint(tm, ti.un.col0 + b * kUBoxCols, ti.m0, w_base + stage * kUWStage + b * kUBoxBytes, pol);
                        bulk_commit();
                    }
                    bulk_wait_read<0>();
                    mbar_arrive(&empty[stage]);
                    ti.next(p);
                }
                bulk_wait_all<0>();
                tl_stamp(tl, 6);
            }
        } else {
            // ============ epilogue warps: group g = warp / 4 takes the tiles with it % 2 == g (TMEM lane quarter =
            // warp % 4).  Sharing every tile between the groups (64 columns each) halves a tile's latency at the
            // phase boundaries but slows the steady state by 5 % (twice the atomics): measured, not kept. ============
            const int group = warp >> 2, quarter = warp & 3;
            const int row_in_tile = quarter * 32 + lane;
            unsigned char* slab = sm + L::off_slab;
            float* xs_all = reinterpret_cast<float*>(sm + L::off_xs);
            UmmaIter ti;
            ti.init(p, unit_cache);
            if (ti.valid(p)) {
                // (programmatic dependent launch: the wait for the previous kernel sits in the first enter_phase, after
                //  this CTA's first slab has been staged and its first MMAs issued -- they only need the factors)
                bool pdl_pending = GEMV && mp.pdl;
                float x_inv = 1.0f, in_scale = 1.0f;
                bool tl_first = false;
                int cur_phase = -1, phase_j0 = 0, published = 0;
                // entering a phase: previous phase published by every CTA, then the input vector
                auto enter_phase = [&](int ph) {
                    const GemvParams& g = mp.gv[ph];
                    if (pdl_pending) {
                        pdl_pending = false;
                        pdl_wait();
                        if (tid == 0) {
                            pdl_launch_dependents();
                            tl_stamp(tl, 3);
                        }
                    }
                    if (tid == 0) tl_stamp(tl, 8 + 4 * ph);
                    if (ph > 0) {
                        if (tid == 0) {
                            // (a reduced phase: the CTAs of EVERY rank report on this rank's counter)
                            const bool reduced = PEERS && mp.n_peers > 0 && ((mp.reduce_mask >> (ph - 1)) & 1);
                            const int target = (int)gridDim.x * (reduced ? mp.n_peers : 1);
                            const long long t0 = clock64();
                            int seen;
                            do {
                                if (PEERS && mp.n_peers > 0)
                                    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(seen) : "l"(mp.phase_done + ph - 1) : "memory");
                                else
                                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(mp.phase_done + ph - 1) : "memory");
                                if (seen >= target) break;
                                const long long waited = clock64() - t0;
                                if (waited > (1ll << 32)) {
                                    if (p.err_flag) atomicExch(p.err_flag, AF_ECUDA);
                                    break;
                                }
                                // (an error already raised -- an earlier launch's timeout, a rank that gave up -- ends later waits
                                //  after ~2 ms instead of ~2 s each: a dead peer fails the step in seconds, not minutes)
                                if (waited > (1ll << 22) && p.err_flag && *reinterpret_cast<volatile int*>(p.err_flag) != 0) break;
                            } while (true);
                        }
                        named_bar_sync(1, kUEpi);
                    }
                    if (tid == 0) tl_stamp(tl, 9 + 4 * ph);
                    x_inv = 1.0f;
                    in_scale = g.inv_in ? __ldcg(g.inv_in) : 1.0f;
                    phase_j0 = ti.j;
                    // strips of this CTA's units of the phase: thread t -> column t % 128 of slots t / 128 and t / 128 + 2
                    float xr_h[2], xr_w[2];
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2) {
                        const int slot = (tid >> 7) + 2 * k2;
                        xr_h[k2] = 0.f;
                        xr_w[k2] = 1.f;
                        const long long uu = (long long)ti.u + (long long)slot * gridDim.x;
                        if (uu < p.n_units) {
                            const UnitDev un2 = ti.fetch(p, ti.j + slot, (int)uu);
                            const int c = un2.col0 + (tid & 127);
                            if (un2.rows > 0 && un2.phase == ph && c < g.x_len) {
                                if (g.prologue == AF_PRO_SILU_MUL) {
                                    xr_h[k2] = gemv_x(g, c, 1.0f, in_scale);
                                } else {
                                    xr_h[k2] = gemv_h(g, c);
                                    if (g.prologue == AF_PRO_RMSNORM || g.prologue == AF_PRO_RMSNORM_DEFERRED) xr_w[k2] = g.norm_w[c];
                                }
                            }
                        }
                    }
                    // the whole-vector pass: every CTA for a plain RMSNorm; CTA 0 alone when the scale is deferred
                    // (or when it only has to materialise h)
                    if (g.prologue == AF_PRO_RMSNORM || ((g.h_out || g.prologue == AF_PRO_RMSNORM_DEFERRED) && blockIdx.x == 0)) {
                        float ss = 0.f;
                        const bool write_h = g.h_out && blockIdx.x == 0;
                        constexpr int kStep = 2 * kUEpi;
                        constexpr int kFly = 8;   // steps of loads in flight: 4096 entries are ONE L2 round trip
                        for (int base = 2 * tid; base < g.x_len; base += kFly * kStep) {
                            float2 hv[kFly];
#pragma unroll
                            for (int u4 = 0; u4 < kFly; ++u4) {
                                const int c = base + u4 * kStep;
                                hv[u4] = make_float2(0.f, 0.f);
                                if (c < g.x_len) {
                                    if (g.acc_in) {
                                        const longlong2 q = __ldcg(reinterpret_cast<const longlong2*>(g.acc_in + c));
                                        hv[u4] = make_float2(fix_to_f32(q.x), fix_to_f32(q.y));
                                    } else {
                                        hv[u4] = __ldcg(reinterpret_cast<const float2*>(g.xin + c));
                                    }
                                    if (g.res) {
                                        const float2 r = __ldcg(reinterpret_cast<const float2*>(g.res + c));
                                        hv[u4].x += r.x;
                                        hv[u4].y += r.y;
                                    }
                                }
                            }
#pragma unroll
                            for (int u4 = 0; u4 < kFly; ++u4) {
                                const int c = base + u4 * kStep;
                                ss = fmaf(hv[u4].x, hv[u4].x, fmaf(hv[u4].y, hv[u4].y, ss));
                                if (write_h && c < g.x_len) *reinterpret_cast<float2*>(g.h_out + c) = hv[u4];
                            }
                        }
                        float* red = reinterpret_cast<float*>(sm + L::off_red);
                        ss = warp_sum(ss);
                        named_bar_sync(1, kUEpi);
                        if (lane == 0) red[warp] = ss;
                        named_bar_sync(1, kUEpi);
                        float tot = 0.f;
#pragma unroll
                        for (int i = 0; i < kUEpiWarps; ++i) tot += red[i];
                        x_inv = rsqrtf(tot / (float)g.x_len + g.eps);
                        if (g.prologue == AF_PRO_RMSNORM_DEFERRED) {
                            if (tid == 0 && g.inv_out) *g.inv_out = x_inv;   // read by the consumer of this launch's outputs
                            x_inv = 1.0f;
                        }
                    }
#pragma unroll
                    for (int k2 = 0; k2 < 2; ++k2) {
                        float v = xr_h[k2];
                        if (g.prologue == AF_PRO_RMSNORM) v *= x_inv * xr_w[k2];
                        else if (g.prologue == AF_PRO_RMSNORM_DEFERRED) v *= xr_w[k2];
                        xs_all[((tid >> 7) + 2 * k2) * kUN + (tid & 127)] = v;
                    }
                    named_bar_sync(1, kUEpi);
                    if (tid == 0) tl_stamp(tl, 10 + 4 * ph);
                    tl_first = true;
                };

                const int rank = seg_of(ti.un).rank;
                const int S = n_blocks * rank;
                uint4 dn_regs[kPrefetchSlab ? NB * 8 * (kUN / 8) / kUEpi : 1];
                if constexpr (kPrefetchSlab) umma_slab_prefetch<NB>(dn_regs, seg_of(ti.un), plan, S, ti.un.col0, tid);
                bool new_unit = true;
                int yoff = 0;
                unsigned long long* acc_out = nullptr;
                const float* xs = nullptr;
                for (int it = 0; ti.valid(p); ++it) {
                    const int stage = it % kSt, buf = it & 1;
                    const uint32_t ph = (it / kSt) & 1, aph = (it >> 1) & 1;
                    if (new_unit) {
                        // every MMA of the previous unit has completed (its last accumulators were read below) and
                        // both groups are here: the slab may be rewritten for this unit
                        named_bar_sync(1, kUEpi);
                        if constexpr (GEMV) {
                            // the phases this CTA has finished (or has no tiles in) are complete on its side: every
                            // epilogue warp issued its atomics before the barrier above -- publish before anything else
                            if (ti.un.phase != cur_phase) {
                                if (tid == 0 && published < ti.un.phase) umma_publish_phases<PEERS>(mp, published, min(ti.un.phase, mp.n_phases - 1));
                                published = ti.un.phase;
                            }
                        }
                        if constexpr (kPrefetchSlab) umma_slab_commit<NB, PC>(slab, dn_regs, plan, S, rank, tid);
                        else if (!(mp.dbg & 128) || it == 0) umma_slab_direct<NB>(slab, seg_of(ti.un), plan, S, ti.un.col0, tid);   // (dbg 128: timing experiment)
                        fence_proxy_async_smem();   // generic writes -> the tensor core's (async proxy) reads
                        __syncwarp();
                        if (lane == 0) mbar_arrive(slab_bar);
                        if constexpr (kPrefetchSlab) {   // start fetching the NEXT unit's DOWN rows; they are committed at its start
                            const UnitDev nu = ti.peek(p);
                            if (nu.rows > 0) umma_slab_prefetch<NB>(dn_regs, seg_of(nu), plan, S, nu.col0, tid);
                        }
                        if constexpr (GEMV) {
                            if (ti.un.phase != cur_phase) {
                                cur_phase = ti.un.phase;
                                enter_phase(cur_phase);
                                acc_out = mp.gv[cur_phase].acc_out;
                            }
                            yoff = mp.seg_yoff[ti.un.seg];
                            const int xslot = ti.j - phase_j0;
                            xs = xslot < kUXSlots ? xs_all + xslot * kUN : nullptr;
                        }
                    }
                    const int m0 = ti.m0, row_end = ti.row_end, col0 = ti.un.col0;
                    new_unit = ti.next(p);
                    if ((it & 1) == group) {
                        const bool probe = GEMV && tl && tl_first && cur_phase == 1 && tid == (it & 1) * 128;   // timeline: first tile of phase 1, one thread per group
                        if (probe) tl_stamp(tl, 26 + 3 * (it & 1));
                        mbar_wait(&full[stage], ph);        // the W tile (TMA) is in shared memory
                        mbar_wait(&acc_full[buf], aph);     // the MMAs of this tile have completed
                        tc_fence_after();
                        if (probe) tl_stamp(tl, 27 + 3 * (it & 1));
                        const uint32_t wrow = w_base + stage * kUWStage + row_in_tile * 128;
                        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + buf * kUN;
                        float y = 0.f;
                        // one 32-column chunk of this thread's row: W + D, round, store back, dot with x
                        auto chunk = [&](const uint32_t (&d)[32], int c4) {
                            const uint32_t wbox = wrow + (c4 >> 1) * kUBoxBytes;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const uint32_t addr = wbox + (((uint32_t)((c4 & 1) * 4 + i) ^ (uint32_t)(row_in_tile & 7)) << 4);
                                uint4 w = lds128(addr);
                                uint32_t in[4] = {w.x, w.y, w.z, w.w}, out[4];
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    out[e] = pack_bf16x2(bf16lo_to_f32(in[e]) + __uint_as_float(d[i * 8 + 2 * e]),
                                                         bf16hi_to_f32(in[e]) + __uint_as_float(d[i * 8 + 2 * e + 1]));
                                sts128(addr, make_uint4(out[0], out[1], out[2], out[3]));
                                if constexpr (GEMV) {
                                    const int c = c4 * 32 + i * 8;
                                    float4 xa, xb;
                                    if (xs) {
                                        xa = *reinterpret_cast<const float4*>(xs + c);
                                        xb = *reinterpret_cast<const float4*>(xs + c + 4);
                                    } else {
                                        const GemvParams& g = mp.gv[cur_phase];
                                        float t[8];
#pragma unroll
                                        for (int e = 0; e < 8; ++e) t[e] = (col0 + c + e < g.x_len) ? gemv_x(g, col0 + c + e, x_inv, in_scale) : 0.f;
                                        xa = make_float4(t[0], t[1], t[2], t[3]);
                                        xb = make_float4(t[4], t[5], t[6], t[7]);
                                    }
                                    // the ROUNDED weights, as a decode after the switch would read them
                                    y = fmaf(bf16lo_to_f32(out[0]), xa.x, y); y = fmaf(bf16hi_to_f32(out[0]), xa.y, y);
                                    y = fmaf(bf16lo_to_f32(out[1]), xa.z, y); y = fmaf(bf16hi_to_f32(out[1]), xa.w, y);
                                    y = fmaf(bf16lo_to_f32(out[2]), xb.x, y); y = fmaf(bf16hi_to_f32(out[2]), xb.y, y);
                                    y = fmaf(bf16lo_to_f32(out[3]), xb.z, y); y = fmaf(bf16hi_to_f32(out[3]), xb.w, y);
                                }
                            }
                        };
#pragma unroll 1
                        for (int c4 = 0; c4 < kUN / 32; ++c4) {
                            uint32_t da[32];
                            tmem_ld32(taddr + c4 * 32, da);
                            tmem_ld_wait();
                            chunk(da, c4);
                        }
                        if (probe) tl_stamp(tl, 28 + 3 * (it & 1));
                        tc_fence_before();
                        fence_proxy_async_smem();   // tile written back -> visible to the TMA store
                        __syncwarp();
                        if (lane == 0) {
                            mbar_arrive(&acc_empty[buf]);
                            mbar_arrive(&computed[stage]);
                        }
                        if constexpr (GEMV) {
                            if (m0 + row_in_tile < row_end) {
                                unsigned long long* dst = acc_out + yoff + m0 + row_in_tile;
                                const unsigned long long v = (unsigned long long)f32_to_fix(y);
                                if (PEERS && mp.n_peers > 0 && ((mp.reduce_mask >> cur_phase) & 1)) {   // row-parallel phase: into every rank's sums
                                    for (int w = 0; w < mp.n_peers; ++w)
                                        atomicAdd_system(reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(dst) + mp.peer_off[w]), v);
                                } else {
                                    atomicAdd(dst, v);
                                }
                            }
                            if (tl_first && tid == (it & 1) * 128) tl_stamp(tl, 11 + 4 * cur_phase);
                        }
                    }
                    tl_first = false;
                }
                if (tid == 0) tl_stamp(tl, 7);
                if constexpr (GEMV) {   // the remaining phases of the chain
                    named_bar_sync(1, kUEpi);
                    if (tid == 0) umma_publish_phases<PEERS>(mp, published, umma_phases_to_publish<PEERS>(mp));
                }
            } else if constexpr (GEMV) {
                // a CTA without work still takes part in the phase barriers
                if (tid == 0) umma_publish_phases<PEERS>(mp, 0, umma_phases_to_publish<PEERS>(mp));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kUEpiWarps + 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

}  // namespace af
