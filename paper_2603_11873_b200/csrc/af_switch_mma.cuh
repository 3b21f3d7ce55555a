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
#ifndef AF_W_EARLY
#define AF_W_EARLY 0    /* W fragments of a tile are loaded before its MMAs (1) or after them (0) */
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
constexpr int kMmaThreadsGemv = kMmaThreads + 32;                          // + the reducer warp of the fused GEMV
constexpr int kMmaMaxKS = 4;                      // k-steps of 16 ranks: S <= 64
constexpr int kMmaMaxStages = 12;
constexpr int kStoreDepth = 0;                    // tile stores that may still be reading smem
constexpr int kMmaDefaultStages = 10;
constexpr int kUnitCache = 24;  // unit descriptors of a CTA cached in shared memory
constexpr int kSegCache = 12;   // segments of a chain (4 phases x up to 3 matrices)
constexpr int kXSlots = 4;      // input-vector strips staged per phase (units of one CTA in one phase)

// BA ("block accumulate"): the slab holds the RAW bf16 DOWN rows and the gate is applied to the
// f32 product of each rank-16 step (acc += g * (U_b A_b)) instead of being folded into a hi+lo
// pair -- half the tensor work, one f32 FMA per element per step.  Used when rank % 16 == 0 and
// the stacked rank exceeds 32 (Llama-3-8B: r = 16, s = 64), where the hi/lo form is HMMA-bound.
template <int KS, bool BA = false, bool GEMV = false>
struct MmaLayout {
    static constexpr int s_pad = KS * 16;
    static constexpr int up_stage_bytes = kMR * s_pad * 2;
    static constexpr int down_bytes = (BA ? 1 : 2) * s_pad * kDownPitch * 2;
    // GEMV: per stage, the 16 consumer warps' partial dot products of the tile's 32 rows (f32)
    static constexpr int part_stage_bytes = GEMV ? kMmaWarps * kMR * 4 : 0;
    static constexpr int red_bytes = GEMV ? 128 : 0;  // block reduction scratch of the RMSNorm prologue
    static constexpr int cache_bytes = kUnitCache * (int)sizeof(UnitDev) + (GEMV ? kSegCache * (int)sizeof(SegDev) : 0);
    static constexpr int xs_bytes = GEMV ? kXSlots * kTN * 4 : 0;  // staged input-vector strips of the current phase
    static constexpr int fixed = down_bytes + 3 * 8 * 16 + (int)sizeof(Plan) + red_bytes + cache_bytes + xs_bytes + 1024 /*alignment slack*/ + 256;
    static constexpr int by_smem = (227 * 1024 - fixed) / (kWStageBytes + up_stage_bytes + part_stage_bytes);
    static constexpr int stages = by_smem < kMmaMaxStages ? by_smem : kMmaMaxStages;
    // offsets from the 1024-aligned base
    static constexpr int off_w = 0;
    static constexpr int off_up = off_w + stages * kWStageBytes;
    static constexpr int off_part = off_up + stages * up_stage_bytes;
    static constexpr int off_down = off_part + stages * part_stage_bytes;
    static constexpr int off_bar = off_down + down_bytes;          // full[16], computed[16], empty[16]
    static constexpr int off_plan = off_bar + 3 * 8 * 16;
    static constexpr int off_red = (off_plan + (int)sizeof(Plan) + 15) & ~15;
    static constexpr int off_units = off_red + red_bytes;
    static constexpr int off_segs = off_units + kUnitCache * (int)sizeof(UnitDev);
    static constexpr int off_xs = (off_segs + (GEMV ? kSegCache * (int)sizeof(SegDev) : 0) + 15) & ~15;
    static constexpr int total = off_xs + xs_bytes + 1024 /*alignment slack*/;
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
// (not volatile: a pure register operation the compiler may interleave with its neighbours)
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// mbarrier / shared-store forms that take the 32-bit shared address directly (computed once per
// unit of work instead of being re-derived from a generic pointer at every use)
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_shared_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
// 1-D bulk copy global -> smem, completes on bar (bytes % 16 == 0, both sides 16-byte aligned).
__device__ __forceinline__ void bulk_load_1d(uint32_t smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// W is touched once per token and is 100x larger than L2: its tiles are loaded and stored with an
// evict-first policy so that the stream does not push out what IS reused -- the selected experts'
// factors (re-read by every column strip), the activation vectors, the accumulators, the code.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(uint32_t smem_dst, const void* tmap, int c0, int c1, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;"
        ::"r"(smem_dst), "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const void* tmap, int c0, int c1, uint32_t smem_src, uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(tmap),
                 "r"(c0), "r"(c1), "r"(smem_src), "l"(pol)
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

// Fixed-point accumulators of the fused GEMV: a row's partial dot products (one per 256-column
// strip, produced by different CTAs) are added with 64-bit INTEGER atomics, so the sum does not
// depend on the order the CTAs arrive in -- the result is deterministic, unlike f32 atomics.
// value = acc * 2^-AF_FIX_SHIFT; resolution 9e-13, range +-8.4e6.
__device__ __forceinline__ float fix_to_f32(long long q) { return __ll2float_rn(q) * (1.0f / (float)(1ll << AF_FIX_SHIFT)); }
__device__ __forceinline__ long long f32_to_fix(float v) { return __float2ll_rn(v * (float)(1ll << AF_FIX_SHIFT)); }

// The GEMV fused into the switch (switch_mma_kernel<..., GEMV = true>): while a tile of W is in
// registers, freshly updated and rounded to bf16, it is also multiplied with the input vector of
// the projection -- the decode forward (model.py:367-368) reads no weight a second time.
//   h[c] = (res ? res[c] : 0) + (acc_in ? fix(acc_in[c]) : xin[c])
//   x[c] = h[c]                                   prologue NONE
//        = h[c] * rsqrt(mean(h^2) + eps) * norm_w prologue RMSNORM
//        = silu(a[c]) * a[x_len + c]              prologue SILU_MUL (a = the un-residualed input)
//   acc_out[seg_yoff[seg] + row] += fix(sum_c Wnew[row][c] * x[c])   per 256-column strip
struct GemvParams {
    const float* xin;
    const long long* acc_in;
    const float* res;
    float* h_out;                  // optional: CTA 0 materialises h (the residual stream)
    const float* norm_w;
    float eps;
    int prologue;
    int x_len;                     // d_in of the group
    unsigned long long* acc_out;
    // Deferred RMSNorm (AF_PRO_RMSNORM_DEFERRED, tcgen05 kernel): the scale rsqrt(mean(h^2) + eps) factors out of
    // the GEMV, so only CTA 0 reads the whole vector (and writes the scale to inv_out); everyone else starts on
    // x' = h * norm_w at once.  The launch's outputs are then unscaled: their consumer multiplies by the scale
    // (inv_in of the SiLU phase that follows, `scale` of af_attn_decode_fix).
    float* inv_out;
    const float* inv_in;           // scale of THIS phase's input accumulators (NULL = 1)
};

// A launch may chain up to kMaxPhases projections whose inputs depend on each other's outputs
// (o -> gate|up -> down -> next layer's q|k|v): the weight stream of phase p+1 never waits -- its
// tiles fill the shared-memory ring while the consumers sit at the phase boundary -- only the
// GEMV input does: consumers spin on a device counter that every CTA's storer bumps once its
// last partial sums of phase p are out (a grid barrier the producers do not take part in).
constexpr int kMaxPhases = 4;

struct MmaParams {
    SwitchParams base;
    GemvParams gv[kMaxPhases];
    int n_phases;
    int* phase_done;               // [n_phases - 1] counters, zeroed by the caller per launch
    const int* seg_yoff;           // per table segment: first row of its slice of its phase's acc_out
    int chain_segs[kSegCache];     // table ids of the chain's segments (UnitDev::slot indexes this list)
    int n_chain_segs;
    int pdl;                       // launched with programmatic stream serialization
    // optional timeline probe (af_set_timeline): [gridDim.x][kTlSlots] globaltimer stamps of this launch
    unsigned long long* timeline;
    int mixed_rank;                // the table's segments do not all have the same rank
    int dbg;                       // bit 8 / 16: L2 evict-first hint on the W loads / stores (on by default; the env
                                   // AF_DBG flips bits for A/B runs; AF_DBG=4: plain switch kernel on a group's schedule)
    const CUtensorMap* tmaps_ld;   // per segment: 32 x 64 swizzled box on the source (live or pristine)
    const CUtensorMap* tmaps_st;   // per segment: the same box shape on the live matrix
    const CUtensorMap* tmaps_up;   // per segment: UP bank as [N * d_out][rank], box 32 rows x rank, swizzle = row bytes
                                   // (used when rank is 16 / 32 / 64: 32-byte+ rows would bank-conflict unswizzled)
    int up_swizzle_ok;             // 0: always plain bulk copies for UP (A/B switch, env AF_UP_SWIZZLE=0)
    int n_stages;                  // ring depth actually used (<= MmaLayout<KS>::stages)
    int store_depth;               // tile stores that may still be reading shared memory (0..3)
    // Tensor parallelism without a collective between the launches (af_group_set_peers, tcgen05 kernel): the
    // fixed-point accumulators and the phase counters live in a buffer every rank maps at
    // (own address + peer_off[w]).  A phase in reduce_mask (row-parallel: o, down) adds its partial sums into EVERY
    // rank's accumulators and is published on every rank's counter, so the next phase starts on the all-reduced
    // vector when gridDim.x * n_peers CTAs have reported -- integer adds, so the sum is exact in any order.
    int n_peers;                   // 0 = single rank (no peer traffic); peer_off[] includes this rank (offset 0)
    int reduce_mask;               // bit ph: phase ph pushes to the peers
    long long peer_off[8];
};

// Gated DOWN slab for one unit: rows [0, S) hold hi(g*a), rows [s_pad, s_pad+S) hold lo; the
// padding rows up to s_pad are zero.  Staging is split in two so the global-load latency hides
// under a whole unit of tiles: down_prefetch() issues this thread's 16-byte loads of the NEXT
// unit's DOWN rows into registers, down_commit() folds the gate (one f32 multiply,
// adapters.py:202), splits into bf16 hi + lo and writes the slab.
// q / r and q % r for the (usually power-of-two) rank: these sit on the per-unit serial path of
// every consumer thread, where a generic integer division costs ~40 dependent instructions.
__device__ __forceinline__ void rank_divmod(int q, int r, int& quo, int& rem) {
    if ((r & (r - 1)) == 0) {
        quo = q >> (31 - __clz(r));
        rem = q & (r - 1);
    } else {
        quo = q / r;
        rem = q % r;
    }
}

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
        // predicated load inside one asm block: nothing consumes the value here, so the thread does
        // not wait for it (a C++ `zero; if (ok) load` becomes load + select, which does)
        const bool ok = q < S && col0 + c < sg.d_in;
        const int qq = ok ? q : 0;
        int b, qr;
        rank_divmod(qq, r, b, qr);
        const __nv_bfloat16* src = base + (long long)plan.expert[b] * sg.down_estride + (long long)qr * sg.ld_down + col0 + c;
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

template <int KS, bool BA>
__device__ __forceinline__ void down_commit(unsigned char* down_smem, const uint4 (&regs)[KS], int rank, const Plan& plan,
                                            int S, int tid) {
    constexpr int s_pad = KS * 16;
    constexpr int chunks_per_row = kTN / 8;
#pragma unroll
    for (int j = 0; j < KS; ++j) {
        const int i = tid + j * kMmaConsumers;
        const int q = i / chunks_per_row;
        const int c = (i % chunks_per_row) * 8;
        if constexpr (BA) {  // raw rows; padding rows are zero (regs were zero-filled by the prefetch)
            *reinterpret_cast<uint4*>(down_smem + ((size_t)q * kDownPitch + c) * 2) = regs[j];
            continue;
        }
        uint4 hi = make_uint4(0u, 0u, 0u, 0u), lo = hi;
        if (q < S) {
            int wb, wr;
            rank_divmod(q, rank, wb, wr);
            const float w = plan.weight[wb];
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

// Tile walk of the tensor-path kernels: as TileIterT<kMR>, but the CTA's first kUnitCache unit
// descriptors come from shared memory (copied once at kernel start).  Under load a global read
// costs ~2 us; a unit change used to pay two of them in a row (unit, then its segment).
struct MmaIter {
    int j, u, m0, row_end;
    UnitDev un;
    const UnitDev* cache;
    __device__ __forceinline__ bool valid(const SwitchParams& p) const { return u < p.n_units; }
    __device__ __forceinline__ UnitDev fetch(const SwitchParams& p, int jj, int uu) const {
        return jj < kUnitCache ? cache[jj] : p.units[uu];
    }
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
        m0 += kMR;
        if (m0 < row_end) return false;
        u += gridDim.x;
        ++j;
        load_unit(p);
        return true;
    }
    // the unit after the current one (rows == 0: none)
    __device__ __forceinline__ UnitDev peek(const SwitchParams& p) const {
        const int un2 = u + gridDim.x;
        if (un2 >= p.n_units) return UnitDev{0, 0, 0, 0, 0, 0};
        return fetch(p, j + 1, un2);
    }
};

// UP rows of 32 / 64 / 128 bytes are fetched through a swizzled 2-D tensor map (swizzle span =
// row bytes) so that the A-fragment ldmatrix of 8 consecutive rows is bank-conflict free; 16-byte
// rows (rank 8) are conflict free as they are and use plain 1-D bulk copies.
__host__ __device__ __forceinline__ bool up_swizzled(int rank) { return rank == 16 || rank == 32 || rank == 64; }

// Warp roles (all walk the same static tile sequence):
//   warps 0..15  consumers: wait full[stage] -> W + U.(hi+lo) in place in smem -> arrive computed[stage]
//   W producers  (kWProd warps, 1 thread each): wait empty[stage] -> TMA loads of their W boxes
//   UP producer  (1 warp, 1 thread): wait empty[stage] -> bulk copies of the selected UP blocks
//   storers      (kStorers warps, 1 thread each): wait computed[stage] -> TMA stores of their
//                boxes; a stage goes back to the producers once every storer's stores have read
//                shared memory (store_depth newer stores may still be draining)
// ---- pieces of the fused GEMV (GEMV = true) ----

// Timeline probe slots (nanoseconds of %globaltimer), one row per CTA:
//   0 entry | 1 plan ready | 2 first slab staged | 3 pdl_wait passed | 4 first W load issued |
//   5 last W load issued | 6 storer done | 7 consumers done |
//   8 + 4 * phase: barrier wait begins | +1 barrier passed | +2 prologue done | +3 first tile of the phase computed
constexpr int kTlSlots = 8 + 4 * 4 + 2 + 6 + 4 + 6;  // [36..41]: cycles spent waiting, per role  // + [24] = %smid; [26..31]: first unit change inside phase 1
// mbarrier wait that adds the cycles it blocked to `acc` when the timeline probe is on
__device__ __forceinline__ void mbar_wait_timed(uint64_t* bar, uint32_t parity, bool on, long long& acc) {
    if (on) {
        const long long t0 = clock64();
        mbar_wait(bar, parity);
        acc += clock64() - t0;
    } else {
        mbar_wait(bar, parity);
    }
}
__device__ __forceinline__ void tl_put(unsigned long long* tl, int slot, long long v) {
    if (tl) tl[(size_t)blockIdx.x * kTlSlots + slot] = (unsigned long long)v;
}
__device__ __forceinline__ void tl_stamp(unsigned long long* tl, int slot) {
    if (tl) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tl[(size_t)blockIdx.x * kTlSlots + slot] = t;
    }
}

// One element of the un-normalised input h (see GemvParams).
// (inputs may have been produced by other CTAs earlier in this very launch: read through L2)
__device__ __forceinline__ float gemv_h(const GemvParams& g, int c) {
    float h = g.acc_in ? fix_to_f32(__ldcg(g.acc_in + c)) : __ldcg(g.xin + c);
    if (g.res) h += __ldcg(g.res + c);
    return h;
}
// One element of the projection's input vector x; inv = rsqrt(mean(h^2) + eps) for RMSNORM.
// in_scale: the deferred RMSNorm scale of the launch that produced acc_in (1 when there is none).
__device__ __forceinline__ float gemv_x(const GemvParams& g, int c, float inv, float in_scale = 1.0f) {
    if (g.prologue == AF_PRO_SILU_MUL) {
        const float a = in_scale * (g.acc_in ? fix_to_f32(__ldcg(g.acc_in + c)) : __ldcg(g.xin + c));
        const float b = in_scale * (g.acc_in ? fix_to_f32(__ldcg(g.acc_in + g.x_len + c)) : __ldcg(g.xin + g.x_len + c));
        return a / (1.0f + expf(-a)) * b;
    }
    float h = gemv_h(g, c);
    if (g.prologue == AF_PRO_RMSNORM) h *= inv * g.norm_w[c];
    else if (g.prologue == AF_PRO_RMSNORM_DEFERRED) h *= g.norm_w[c];
    return h;
}
// B fragment (k16 x n8, col-major) of the input vector for this warp's 16 columns: column n = 0
// carries bf16 hi(x), n = 1 carries lo = x - hi (x is reproduced to 2^-17 relative), the other six
// columns are zero.  Lane j < 16 evaluates x at column col0 + 16 * warp + j.
// `xs` != nullptr: the strip was staged in shared memory at phase entry (the usual case).
__device__ __forceinline__ void gemv_x_fragment(const GemvParams& g, const float* xs, int col0, int warp, int lane, float inv,
                                                uint32_t& xb0, uint32_t& xb1) {
    float xv = 0.f;
    const int c = col0 + warp * 16 + (lane & 15);
    if (xs) {
        if (lane < 16) xv = xs[warp * 16 + lane];
    } else if (lane < 16 && c < g.x_len) {
        xv = gemv_x(g, c, inv);
    }
    const float hi = __bfloat162float(__float2bfloat16_rn(xv));
    const float lo = xv - hi;
    const int t2 = (lane & 3) * 2, n = lane >> 2;
    const float h0 = __shfl_sync(0xffffffffu, hi, t2), h1 = __shfl_sync(0xffffffffu, hi, t2 + 1);
    const float h2 = __shfl_sync(0xffffffffu, hi, t2 + 8), h3 = __shfl_sync(0xffffffffu, hi, t2 + 9);
    const float l0 = __shfl_sync(0xffffffffu, lo, t2), l1 = __shfl_sync(0xffffffffu, lo, t2 + 1);
    const float l2 = __shfl_sync(0xffffffffu, lo, t2 + 8), l3 = __shfl_sync(0xffffffffu, lo, t2 + 9);
    xb0 = n == 0 ? pack_bf16x2(h0, h1) : (n == 1 ? pack_bf16x2(l0, l1) : 0u);
    xb1 = n == 0 ? pack_bf16x2(h2, h3) : (n == 1 ? pack_bf16x2(l2, l3) : 0u);
}

// TL: timeline probe compiled in (af_set_timeline); the production instantiations carry none of it.
template <int KS, bool BA, bool GEMV, bool TL = false>
__global__ void __launch_bounds__(GEMV ? kMmaThreadsGemv : kMmaThreads, 1) switch_mma_kernel(const __grid_constant__ MmaParams mp) {
    using L = MmaLayout<KS, BA, GEMV>;
    constexpr int kSt = L::stages < kMmaDefaultStages ? L::stages : kMmaDefaultStages;
    extern __shared__ unsigned char smem_dyn[];
    const SwitchParams& p = mp.base;
    // 128-byte swizzle needs 1024-byte aligned boxes
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::off_bar);
    uint64_t* computed = full + 16;
    uint64_t* empty = full + 32;
    Plan& plan = *reinterpret_cast<Plan*>(sm + L::off_plan);
    UnitDev* unit_cache = reinterpret_cast<UnitDev*>(sm + L::off_units);
    SegDev* seg_cache = reinterpret_cast<SegDev*>(sm + L::off_segs);
    const int tid = threadIdx.x;
    // descriptor caches (one global round trip, concurrent with the plan build below)
    if (tid >= 32 && tid < 32 + kUnitCache) {
        const int jj = tid - 32;
        const long long uu = (long long)blockIdx.x + (long long)jj * gridDim.x;
        unit_cache[jj] = uu < p.n_units ? p.units[uu] : UnitDev{0, 0, 0, 0, 0, 0};
    }
    if constexpr (GEMV) {
        if (tid >= 64 && tid < 64 + mp.n_chain_segs) seg_cache[tid - 64] = p.segs[mp.chain_segs[tid - 64]];
    }
    // the UP ring starts as zeros (see need_mask)
    for (int i = tid * 16; i < kSt * L::up_stage_bytes; i += (int)blockDim.x * 16)
        *reinterpret_cast<uint4*>(sm + L::off_up + i) = make_uint4(0u, 0u, 0u, 0u);
    // descriptor of a unit's segment
    auto seg_of = [&](const UnitDev& un) -> SegDev { return GEMV ? seg_cache[un.slot] : p.segs[un.seg]; };

    if (tid == 0) {
        if constexpr (GEMV) {
            if constexpr (TL) tl_stamp(mp.timeline, 0);
            if (mp.timeline) {
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                mp.timeline[(size_t)blockIdx.x * kTlSlots + 24] = smid;
            }
        }
        for (int s = 0; s < kSt; ++s) {
            mbar_init(&full[s], kWProd + 1);
            mbar_init(&computed[s], kMmaWarps);
            mbar_init(&empty[s], kStorers + (GEMV ? 1 : 0));
        }
        fence_mbar_init();
        if (!p.plan_dev) {
            if (p.use_dev)
                build_plan(plan, p.from_pristine ? nullptr : p.prev_dev, p.cur_dev, p.scale, false, p.n_experts_limit);
            else
                plan = p.host_plan;
            if (!plan_usable(p, plan, p.prev_dev, p.cur_dev)) plan.n_blocks = -1;
        }
        if constexpr (GEMV) if constexpr (TL) tl_stamp(mp.timeline, 1);
    }
    if (p.plan_dev) {  // prebuilt by af_plan_build: one global round trip, concurrent with the barrier setup
        constexpr int kWords = (int)(sizeof(Plan) / 4);
        if (tid >= 128 && tid < 128 + kWords)
            reinterpret_cast<int*>(&plan)[tid - 128] = reinterpret_cast<const int*>(p.plan_dev)[tid - 128];
    }
    __syncthreads();
    const int n_blocks = plan.n_blocks;
    if (n_blocks < 0) return;                       // unusable decision: flagged, nothing touched
    // unchanged decision: nothing to move (the fused GEMV still has to stream W, but stores nothing)
    const bool store_w = n_blocks > 0 || p.from_pristine;
    if (!GEMV && !store_w) return;

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
            const uint64_t pol = l2_evict_first_policy();
            long long waited = 0;
            MmaIter ti;
            ti.init(p, unit_cache);
            for (int it = 0; ti.valid(p); ++it) {
                const int stage = it % kSt;
                const uint32_t ph = (it / kSt) & 1;
                mbar_wait_timed(&empty[stage], ph ^ 1, TL && mp.timeline, waited);
                int mine = 0;
#pragma unroll
                for (int j = 0; j < kMine; ++j) mine += (who + j * kWProd < kBoxes) ? 1 : 0;
                mbar_expect_tx(&full[stage], mine * kBoxBytes);
                if constexpr (GEMV) {
                    if (who == 0 && it == 0) if constexpr (TL) tl_stamp(mp.timeline, 4);
                }
                const CUtensorMap* tm = mp.tmaps_ld + ti.un.seg;
#pragma unroll
                for (int j = 0; j < kMine; ++j) {
                    const int b = who + j * kWProd;
                    if (b < kBoxes) {
                        if (mp.dbg & 8)
                            tma_load_2d_hint(w_base + stage * kWStageBytes + b * kBoxBytes, tm, ti.un.col0 + b * kBoxCols, ti.m0,
                                             &full[stage], pol);
                        else
                            tma_load_2d_addr(w_base + stage * kWStageBytes + b * kBoxBytes, tm, ti.un.col0 + b * kBoxCols, ti.m0,
                                             &full[stage]);
                    }
                }
                ti.next(p);
            }
            if constexpr (GEMV) {
                if (who == 0) {
                    if constexpr (TL) tl_stamp(mp.timeline, 5);
                    if constexpr (TL) tl_put(mp.timeline, 37, waited);
                }
            }
        }
        return;
    }
    if (warp == kMmaWarps + kWProd) {
        // ============ UP producer: one 1-D bulk copy per selected expert block ============
        if (lane == 0) {
            MmaIter ti;
            ti.init(p, unit_cache);
            SegDev sg;
            int cur_seg = -1;
            for (int it = 0; ti.valid(p); ++it) {
                const int stage = it % kSt;
                const uint32_t ph = (it / kSt) & 1;
                if (ti.un.seg != cur_seg) {
                    cur_seg = ti.un.seg;
                    sg = seg_of(ti.un);
                }
                const int rows_here = min(kMR, sg.d_out - ti.m0);
                mbar_wait(&empty[stage], ph ^ 1);
                if (mp.up_swizzle_ok && up_swizzled(sg.rank)) {
                    // 2-D boxes (32 rows x rank) through the swizzled tensor map: always whole boxes
                    const uint32_t box_bytes = (uint32_t)kMR * sg.rank * 2;
                    mbar_expect_tx(&full[stage], n_blocks * box_bytes);
                    const CUtensorMap* tm = mp.tmaps_up + ti.un.seg;
                    for (int b = 0; b < n_blocks; ++b)
                        tma_load_2d_addr(up_base + stage * L::up_stage_bytes + b * box_bytes, tm, 0,
                                         plan.expert[b] * sg.d_out + ti.m0, &full[stage]);
                } else {
                    const uint32_t up_blk_bytes = (uint32_t)rows_here * sg.rank * 2;
                    mbar_expect_tx(&full[stage], n_blocks * up_blk_bytes);
                    const __nv_bfloat16* upb = reinterpret_cast<const __nv_bfloat16*>(sg.up);
                    for (int b = 0; b < n_blocks; ++b)
                        bulk_load_1d(up_base + stage * L::up_stage_bytes + b * (kMR * sg.rank * 2),
                                     upb + (long long)plan.expert[b] * sg.up_estride + (long long)ti.m0 * sg.rank,
                                     up_blk_bytes, &full[stage]);
                }
                ti.next(p);
            }
        }
        return;
    }
    if (warp > kMmaWarps + kWProd && warp <= kMmaWarps + kWProd + kStorers) {
        // ============ storers: boxes back to global, then hand the stage back ============
        if (lane == 0) {
            const int who = warp - (kMmaWarps + kWProd + 1);
            constexpr int kMine = (kBoxes + kStorers - 1) / kStorers;
            const uint64_t pol = l2_evict_first_policy();
            long long waited = 0, waited_read = 0;
            MmaIter ti;
            ti.init(p, unit_cache);
            int it = 0;
            for (; ti.valid(p); ++it) {
                const int stage = it % kSt;
                const uint32_t ph = (it / kSt) & 1;
                mbar_wait_timed(&computed[stage], ph, TL && mp.timeline, waited);
                if (store_w) {
                    const CUtensorMap* tm = mp.tmaps_st + ti.un.seg;
#pragma unroll
                    for (int j = 0; j < kMine; ++j) {
                        const int b = who + j * kStorers;
                        if (b < kBoxes)
                        {
                            if (mp.dbg & 16)
                                tma_store_2d_hint(tm, ti.un.col0 + b * kBoxCols, ti.m0, w_base + stage * kWStageBytes + b * kBoxBytes, pol);
                            else
                                tma_store_2d_addr(tm, ti.un.col0 + b * kBoxCols, ti.m0, w_base + stage * kWStageBytes + b * kBoxBytes);
                        }
                    }
                    bulk_commit();
                }
                // the stores of tile it - depth have drained their stage: hand it back
                const int depth = mp.store_depth;
                const long long tr0 = (TL && mp.timeline) ? clock64() : 0;
                if (depth <= 0) bulk_wait_read<0>();
                else if (depth == 1) bulk_wait_read<1>();
                else if (depth == 2) bulk_wait_read<2>();
                else bulk_wait_read<3>();
                if (TL && mp.timeline) waited_read += clock64() - tr0;
                if (it >= depth) mbar_arrive(&empty[(it - depth) % kSt]);
                ti.next(p);
            }
            bulk_wait_all<0>();  // global writes complete before the CTA retires
            if constexpr (GEMV) {
                if constexpr (TL) tl_stamp(mp.timeline, 6);
                if constexpr (TL) tl_put(mp.timeline, 38, waited);
                if constexpr (TL) tl_put(mp.timeline, 39, waited_read);
            }
        }
        return;
    }
    if constexpr (GEMV) {
        if (warp > kMmaWarps + kWProd + kStorers) {
            // ============ reducer (GEMV only): adds the 16 consumer warps' partial dot products of a
            // tile in a fixed order and accumulates the 32 row sums into the phase's fixed-point
            // vector; publishes a finished phase of a chain.  Its own warp, so that neither the
            // stores nor the consumers wait for the shared-memory reads and the atomics. ============
            MmaIter ti;
            ti.init(p, unit_cache);
            int cur_seg = -1, yoff = 0, cur_phase = 0;
            unsigned long long* acc_out = nullptr;
            // phases [from, to) of the chain are complete on this CTA: publish (the atomics of every
            // lane are ordered before lane 0's fence by the __syncwarp)
            auto phases_done = [&](int from, int to) {
                __syncwarp();
                if (lane == 0 && from < to) {
                    __threadfence();
                    for (int ph = from; ph < to && ph < mp.n_phases - 1; ++ph) atomicAdd(mp.phase_done + ph, 1);
                }
            };
            if (mp.pdl) pdl_wait();  // acc_out may still be read by an earlier kernel of the chain
            for (int it = 0; ti.valid(p); ++it) {
                const int stage = it % kSt;
                const uint32_t ph = (it / kSt) & 1;
                // publish finished phases BEFORE waiting for the next phase's first tile: its
                // consumers are waiting for exactly this
                if (ti.un.phase != cur_phase) {
                    phases_done(cur_phase, ti.un.phase);
                    cur_phase = ti.un.phase;
                }
                if (ti.un.seg != cur_seg) {
                    cur_seg = ti.un.seg;
                    yoff = mp.seg_yoff[cur_seg];
                    acc_out = mp.gv[cur_phase].acc_out;
                }
                mbar_wait(&computed[stage], ph);
                const float* part = reinterpret_cast<const float*>(sm + L::off_part + stage * L::part_stage_bytes);
                float sum = 0.f;
#pragma unroll
                for (int w = 0; w < kMmaWarps; ++w) sum += part[w * kMR + lane];
                if (ti.m0 + lane < ti.row_end)
                    atomicAdd(acc_out + yoff + ti.m0 + lane, (unsigned long long)f32_to_fix(sum));
                __syncwarp();  // every lane has read the stage's partials before it is handed back
                if (lane == 0) mbar_arrive(&empty[stage]);
                ti.next(p);
            }
            phases_done(cur_phase, mp.n_phases - 1);
            return;
        }
    }

    // ================================ consumers ====================================
    const int mi = lane >> 3, rr = lane & 7;       // ldmatrix: lane supplies row rr of matrix mi
    const int wbox = warp >> 2;                    // this warp: 16 columns = chunks (warp & 3) * 2 + {0, 1} of box wbox
    const int wchunk = (warp & 3) * 2 + (mi >> 1);
    const int ncol = warp * 16 + (mi >> 1) * 8;    // slab column this lane addresses
    unsigned char* down_smem = sm + L::off_down;
    const uint32_t down_base = smem_u32(down_smem);

    MmaIter ti;
    ti.init(p, unit_cache);
    if (!ti.valid(p)) return;
    SegDev sg = seg_of(ti.un);
    int S = n_blocks * sg.rank;
    uint4 dn_regs[KS];
    down_prefetch<KS>(dn_regs, sg, plan, S, ti.un.col0, tid);
    down_commit<KS, BA>(down_smem, dn_regs, sg.rank, plan, S, tid);
    named_bar_sync(1, kMmaConsumers);  // first slab visible
    // ---- GEMV: everything above (and the W ring the producers are filling) is independent of the
    //      previous kernel; the input vector is not ----
    float x_inv = 1.0f;
    uint32_t xb0 = 0u, xb1 = 0u;
    int cur_phase = -1, phase_j0 = 0;
    bool tl_first_tile = false, tl_probe = false, tl_probe_done = false;
    long long cons_waited = 0;
    const long long cons_t0 = TL ? clock64() : 0;
    if constexpr (GEMV) {
        if (tid == 0) if constexpr (TL) tl_stamp(mp.timeline, 2);
        if (mp.pdl) {
            pdl_wait();
            // the dependent may start (its own pre-wait part reads nothing this chain writes later
            // than one kernel back); triggered after the wait so the chain stays one kernel deep
            if (tid == 0) pdl_launch_dependents();
        }
        if (tid == 0) if constexpr (TL) tl_stamp(mp.timeline, 3);
    }
    // Entering phase ph of the chain: wait until every CTA has published its partial sums of phase
    // ph - 1, then the prologue over the whole input vector (RMSNorm scale, residual stream out).
    auto enter_phase = [&](int ph) {
        const GemvParams& g = mp.gv[ph];
        if (tid == 0) if constexpr (TL) tl_stamp(mp.timeline, 8 + 4 * ph);
        if (ph > 0) {
            if (tid == 0) {
                const int target = (int)gridDim.x;
                const long long t0 = clock64();
                int seen;
                do {
                    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(mp.phase_done + ph - 1) : "memory");
                    if (seen >= target) break;
                    __nanosleep(32);
                    if (clock64() - t0 > (1ll << 32)) {  // ~2 s: never hang the device on a lost CTA
                        if (p.err_flag) atomicExch(p.err_flag, AF_ECUDA);
                        break;
                    }
                } while (true);
            }
            named_bar_sync(1, kMmaConsumers);
        }
        if (tid == 0) if constexpr (TL) tl_stamp(mp.timeline, 9 + 4 * ph);
        x_inv = 1.0f;
        // Input-vector strips of this CTA's units of the phase (at most kXSlots of them) are staged in
        // shared memory now: their loads go out together with the whole-vector pass below -- ONE
        // global round trip (~2 us under load) per phase instead of one more at every unit start.
        phase_j0 = ti.j;
        float xr_h[kXSlots / 2], xr_w[kXSlots / 2];   // thread t: column t % 256 of slots t / 256 and t / 256 + 2
#pragma unroll
        for (int k2 = 0; k2 < kXSlots / 2; ++k2) {
            const int slot = (tid >> 8) + 2 * k2;
            xr_h[k2] = 0.f;
            xr_w[k2] = 1.f;
            const int jj = ti.j + slot;
            const long long uu = (long long)ti.u + (long long)slot * gridDim.x;
            if (uu < p.n_units) {
                const UnitDev un2 = ti.fetch(p, jj, (int)uu);
                const int c = un2.col0 + (tid & 255);
                if (un2.rows > 0 && un2.phase == ph && c < g.x_len) {
                    if (g.prologue == AF_PRO_SILU_MUL) {
                        xr_h[k2] = gemv_x(g, c, 1.0f);
                    } else {
                        xr_h[k2] = gemv_h(g, c);
                        if (g.prologue == AF_PRO_RMSNORM) xr_w[k2] = g.norm_w[c];
                    }
                }
            }
        }
        if (g.prologue == AF_PRO_RMSNORM || (g.h_out && blockIdx.x == 0)) {
            // whole-vector pass, two elements per thread and step, four steps of loads in flight
            float ss = 0.f;
            const bool write_h = g.h_out && blockIdx.x == 0;
            constexpr int kStep = 2 * kMmaConsumers;
            for (int base = 2 * tid; base < g.x_len; base += 4 * kStep) {
                float2 hv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = base + u * kStep;
                    hv[u] = make_float2(0.f, 0.f);
                    if (c < g.x_len) {
                        if (g.acc_in) {
                            const longlong2 q = __ldcg(reinterpret_cast<const longlong2*>(g.acc_in + c));
                            hv[u] = make_float2(fix_to_f32(q.x), fix_to_f32(q.y));
                        } else {
                            hv[u] = __ldcg(reinterpret_cast<const float2*>(g.xin + c));
                        }
                        if (g.res) {
                            const float2 r = __ldcg(reinterpret_cast<const float2*>(g.res + c));
                            hv[u].x += r.x;
                            hv[u].y += r.y;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int c = base + u * kStep;
                    ss = fmaf(hv[u].x, hv[u].x, fmaf(hv[u].y, hv[u].y, ss));
                    if (write_h && c < g.x_len) *reinterpret_cast<float2*>(g.h_out + c) = hv[u];
                }
            }
            float* red = reinterpret_cast<float*>(sm + L::off_red);
            ss = warp_sum(ss);
            named_bar_sync(1, kMmaConsumers);  // the previous phase's readers of red[] are done
            if (lane == 0) red[warp] = ss;
            named_bar_sync(1, kMmaConsumers);
            float tot = 0.f;
#pragma unroll
            for (int i = 0; i < kMmaWarps; ++i) tot += red[i];
            x_inv = rsqrtf(tot / (float)g.x_len + g.eps);
        }
        {
            float* xs = reinterpret_cast<float*>(sm + L::off_xs);
#pragma unroll
            for (int k2 = 0; k2 < kXSlots / 2; ++k2) {
                float v = xr_h[k2];
                if (g.prologue == AF_PRO_RMSNORM) v *= x_inv * xr_w[k2];   // same expression as gemv_x
                xs[((tid >> 8) + 2 * k2) * kTN + (tid & 255)] = v;
            }
            named_bar_sync(1, kMmaConsumers);  // strips visible to every consumer warp
        }
        if (tid == 0) if constexpr (TL) tl_stamp(mp.timeline, 10 + 4 * ph);
        tl_first_tile = true;
    };
    bool new_unit = true;
    constexpr int kHalves = BA ? 1 : 2;
    constexpr int kMT = kMR / 16;
    uint32_t bfr[kHalves][KS][4];
    float gate[KS];  // BA: signed gate of the block each rank-16 step belongs to (0 past the stacked rank)
#pragma unroll
    for (int j = 0; j < KS; ++j) gate[j] = 0.f;
    // per-lane constants of the unit (hoisted out of the tile loop: the integer divisions by the
    // rank and the swizzle arithmetic are paid once per unit, not once per 16 rows)
    const int lrow = (mi & 1) * 8 + rr;                               // row inside an m16 tile this lane addresses
    const uint32_t w_off = lrow * 128 + ((wchunk ^ rr) << 4);         // (row & 7) == rr for every m16 tile
    uint32_t a_off[KS];                                               // A-fragment byte offset inside the UP stage
    uint32_t a_keep_lo[KS], a_keep_hi[KS];                            // (switch-only loop) 0 / ~0: zero the fragment halves past S
    uint32_t a_mt_stride = 0;
    bool need_mask = false;       // the stacked rank does not fill the last rank-16 step: zero the A fragments past it
    int rank_next = sg.rank, S_next = 0;
    bool have_next = false;
    // shared addresses of the ring, advanced with the stage instead of being rebuilt per tile
    const uint32_t w_lane_base = w_base + wbox * kBoxBytes + w_off;
    const uint32_t full_u32 = smem_u32(full), computed_u32 = smem_u32(computed);
    const uint32_t part_lane = smem_u32(sm + L::off_part) + (warp * kMR + (lane >> 2)) * 4;
    int stage = 0;
    uint32_t ph = 0;
    for (; ti.valid(p);) {
        if (new_unit) {
            // B fragments of this unit's slab -> registers (kept for every tile of the unit)
#pragma unroll
            for (int half = 0; half < kHalves; ++half)
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    const int krow = half * L::s_pad + 16 * j + (mi & 1) * 8 + rr;
                    ldmatrix_x4_trans(bfr[half][j], down_base + (krow * kDownPitch + ncol) * 2);
                }
            if constexpr (BA) {
#pragma unroll
                for (int j = 0; j < KS; ++j) gate[j] = (16 * j < S) ? plan.weight[(16 * j) / sg.rank] : 0.f;
            }
            if (TL && tl_probe) tl_stamp(mp.timeline, 33);
            a_mt_stride = 16 * sg.rank * 2;
            // With one rank for the whole table a block's slot in the UP ring never moves, so the slots
            // past the stacked rank keep the zeros the ring was initialised with; only tables that mix
            // ranks can leave another segment's rows there.
            need_mask = mp.mixed_rank && S != KS * 16;
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const int k0 = 16 * j + (mi >> 1) * 8;  // first rank of the 8x8 matrix this lane addresses
                const int kk = k0 < S ? k0 : 0;
                int b, kin;
                rank_divmod(kk, sg.rank, b, kin);
                // 16-byte chunk index inside the row, XOR-swizzled when the block came through the
                // swizzled tensor map (address bits [4..] ^= bits [7..], span = row bytes)
                const int span16 = (mp.up_swizzle_ok && up_swizzled(sg.rank)) ? sg.rank / 8 : 1;  // row bytes / 16
                const int chunk = (kin >> 3) ^ ((lrow / (8 / (span16 > 8 ? 8 : span16))) & (span16 - 1));
                a_off[j] = ((b * kMR + lrow) * sg.rank) * 2 + (chunk << 4);
                a_keep_lo[j] = (16 * j < S) ? 0xffffffffu : 0u;
                a_keep_hi[j] = (16 * j + 8 < S) ? 0xffffffffu : 0u;
            }
            if (TL && tl_probe) tl_stamp(mp.timeline, 34);
            // start fetching the NEXT unit's DOWN rows; they are committed to the slab at its start
            const UnitDev nu = ti.peek(p);
            have_next = nu.rows > 0;
            if (have_next) {
                const SegDev sn = seg_of(nu);
                rank_next = sn.rank;
                S_next = n_blocks * sn.rank;
                down_prefetch<KS>(dn_regs, sn, plan, S_next, nu.col0, tid);
            }
            if (TL && tl_probe) tl_stamp(mp.timeline, 35);
            // The input vector comes LAST: everything above is independent of it, so at a phase
            // boundary it runs while this CTA's own partial sums are still being published and the
            // other CTAs are still arriving.
            if constexpr (GEMV) {
                if (ti.un.phase != cur_phase) {
                    cur_phase = ti.un.phase;
                    enter_phase(cur_phase);
                }
                const int xslot = ti.j - phase_j0;
                const float* xs = xslot < kXSlots ? reinterpret_cast<const float*>(sm + L::off_xs) + xslot * kTN : nullptr;
                gemv_x_fragment(mp.gv[cur_phase], xs, ti.un.col0, warp, lane, x_inv, xb0, xb1);
                if (TL && tl_probe) tl_stamp(mp.timeline, 32);
            }
        }
        new_unit = ti.next(p);

        if (TL && tl_probe) tl_stamp(mp.timeline, 29);
        if constexpr (TL) {
            mbar_wait_timed(&full[stage], ph, mp.timeline != nullptr, cons_waited);
        } else {
            mbar_wait_u32(full_u32 + stage * 8, ph);
        }
        if (TL && tl_probe) tl_stamp(mp.timeline, 30);
        const uint32_t w_stage = w_lane_base + stage * kWStageBytes;
        const uint32_t up_stage = up_base + stage * L::up_stage_bytes;
        if constexpr (!GEMV) {
            // Switch only: one m16 half at a time, W fragment first.  (Measured on one box against
            // the interleaved form below: 4.68 vs 4.83 ms on the Llama-2-7B table -- without the
            // GEMV's extra work the shorter live ranges win; with it the four-chain form does.)
#pragma unroll
            for (int mt = 0; mt < kMT; ++mt) {
                const uint32_t waddr = w_stage + mt * (16 * 128);
                uint32_t wv[4];
                ldmatrix_x4(wv, waddr);
                // A fragments (UP rows); ranks past S are padding and read as 0 (the slab rows are 0 too)
                uint32_t afrag[KS][4];
#pragma unroll
                for (int j = 0; j < KS; ++j) {
                    ldmatrix_x4(afrag[j], up_stage + a_off[j] + mt * a_mt_stride);
                    afrag[j][0] &= a_keep_lo[j];
                    afrag[j][1] &= a_keep_lo[j];
                    afrag[j][2] &= a_keep_hi[j];
                    afrag[j][3] &= a_keep_hi[j];
                }
                float acc[2][4];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
                if constexpr (BA) {
#pragma unroll
                    for (int j = 0; j < KS; ++j) {
                        float pr[2][4] = {};
                        mma_bf16_16816(pr[0], afrag[j], bfr[0][j][0], bfr[0][j][1]);
                        mma_bf16_16816(pr[1], afrag[j], bfr[0][j][2], bfr[0][j][3]);
#pragma unroll
                        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                            for (int e = 0; e < 4; ++e) acc[nt][e] = fmaf(gate[j], pr[nt][e], acc[nt][e]);
                    }
                } else {
                    // same accumulation order as the fused GEMV loop (rank step outer, hi then lo):
                    // both kernels leave bit-identical weights
#pragma unroll
                    for (int j = 0; j < KS; ++j)
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            mma_bf16_16816(acc[0], afrag[j], bfr[half][j][0], bfr[half][j][1]);
                            mma_bf16_16816(acc[1], afrag[j], bfr[half][j][2], bfr[half][j][3]);
                        }
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
        } else {
            // Both m16 halves of the tile advance together: four independent accumulator chains
            // (2 halves x 2 n8 tiles) instead of two, so a dependent HMMA never waits alone.
            uint32_t wv[kMT][4];
    #if AF_W_EARLY
    #pragma unroll
            for (int mt = 0; mt < kMT; ++mt) ldmatrix_x4(wv[mt], w_stage + mt * (16 * 128));   // in flight under the MMAs
    #endif
            float acc[kMT][2][4];
    #pragma unroll
            for (int mt = 0; mt < kMT; ++mt)
    #pragma unroll
                for (int nt = 0; nt < 2; ++nt)
    #pragma unroll
                    for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.f;
    #pragma unroll
            for (int j = 0; j < KS; ++j) {
                // A fragments (UP rows) of rank step j for both halves
                uint32_t afrag[kMT][4];
    #pragma unroll
                for (int mt = 0; mt < kMT; ++mt) ldmatrix_x4(afrag[mt], up_stage + a_off[j] + mt * a_mt_stride);
                if (need_mask) {  // ranks past S are padding: the ring may hold stale data there, read it as 0
                    asm volatile("" ::: "memory");  // keep this a branch: the common case must not pay for the selects
                    const uint32_t keep_lo = (16 * j < S) ? 0xffffffffu : 0u, keep_hi = (16 * j + 8 < S) ? 0xffffffffu : 0u;
    #pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) {
                        afrag[mt][0] &= keep_lo;
                        afrag[mt][1] &= keep_lo;
                        afrag[mt][2] &= keep_hi;
                        afrag[mt][3] &= keep_hi;
                    }
                }
                if constexpr (BA) {
    #pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) {
                        float pr[2][4] = {};
                        mma_bf16_16816(pr[0], afrag[mt], bfr[0][j][0], bfr[0][j][1]);
                        mma_bf16_16816(pr[1], afrag[mt], bfr[0][j][2], bfr[0][j][3]);
    #pragma unroll
                        for (int nt = 0; nt < 2; ++nt)
    #pragma unroll
                            for (int e = 0; e < 4; ++e) acc[mt][nt][e] = fmaf(gate[j], pr[nt][e], acc[mt][nt][e]);
                    }
                } else {
    #pragma unroll
                    for (int half = 0; half < 2; ++half)
    #pragma unroll
                        for (int mt = 0; mt < kMT; ++mt) {
                            mma_bf16_16816(acc[mt][0], afrag[mt], bfr[half][j][0], bfr[half][j][1]);
                            mma_bf16_16816(acc[mt][1], afrag[mt], bfr[half][j][2], bfr[half][j][3]);
                        }
                }
            }
            // W + D, rounded RNE to bf16, written back in place (swizzled smem)
    #if !AF_W_EARLY
    #pragma unroll
            for (int mt = 0; mt < kMT; ++mt) ldmatrix_x4(wv[mt], w_stage + mt * (16 * 128));
    #endif
    #pragma unroll
            for (int mt = 0; mt < kMT; ++mt) {
    #pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    const uint32_t a = wv[mt][nt * 2], b2 = wv[mt][nt * 2 + 1];
                    wv[mt][nt * 2] = pack_bf16x2(bf16lo_to_f32(a) + acc[mt][nt][0], bf16hi_to_f32(a) + acc[mt][nt][1]);
                    wv[mt][nt * 2 + 1] = pack_bf16x2(bf16lo_to_f32(b2) + acc[mt][nt][2], bf16hi_to_f32(b2) + acc[mt][nt][3]);
                }
                stmatrix_x4(w_stage + mt * (16 * 128), wv[mt]);
            }
            if constexpr (GEMV) {
                // the rounded tile is an A fragment as it stands: y[16 rows] = Wnew[16 x 16] . x[16]
                float yv[kMT][4];
    #pragma unroll
                for (int mt = 0; mt < kMT; ++mt) {
    #pragma unroll
                    for (int e = 0; e < 4; ++e) yv[mt][e] = 0.f;
                    mma_bf16_16816(yv[mt], wv[mt], xb0, xb1);
                }
                if ((lane & 3) == 0) {  // columns n = 0 (hi) and n = 1 (lo) of rows lane/4 and lane/4 + 8
                    const uint32_t pa = part_lane + stage * L::part_stage_bytes;
    #pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) {
                        st_shared_f32(pa + mt * 64, yv[mt][0] + yv[mt][1]);
                        st_shared_f32(pa + mt * 64 + 32, yv[mt][2] + yv[mt][3]);
                    }
                }
            }
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the TMA store
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(computed_u32 + stage * 8);
        if (++stage == kSt) {
            stage = 0;
            ph ^= 1;
        }
        if constexpr (TL) {
            if (tl_probe) {
                tl_stamp(mp.timeline, 31);
                tl_probe = false;
            }
            if (tl_first_tile) {
                if (tid == 0) tl_stamp(mp.timeline, 11 + 4 * cur_phase);
                tl_first_tile = false;
            }
        }

        if (new_unit && have_next) {
            const bool probe = TL && tid == 0 && cur_phase == 1 && ti.valid(p) && ti.un.phase == 1 && !tl_probe_done;
            if (probe) tl_stamp(mp.timeline, 26);
            named_bar_sync(1, kMmaConsumers);  // every warp holds its B fragments: the slab may be rewritten
            if (probe) tl_stamp(mp.timeline, 27);
            sg.rank = rank_next;
            S = S_next;
            down_commit<KS, BA>(down_smem, dn_regs, sg.rank, plan, S, tid);
            named_bar_sync(1, kMmaConsumers);  // next slab visible
            if (probe) {
                tl_stamp(mp.timeline, 28);
                tl_probe = true;
                tl_probe_done = true;
            }
        }
    }
    if constexpr (TL) {
        if (tid == 0) {
            tl_stamp(mp.timeline, 7);
            tl_put(mp.timeline, 36, cons_waited);
            tl_put(mp.timeline, 41, clock64() - cons_t0);
        }
    }
}

}  // namespace af
