// af_api.cu -- the C ABI of include/adafuse_b200.h: validation, descriptor tables, TMA maps,
// kernel selection and launches.  No torch types anywhere; every device buffer belongs to the
// caller.  Citations are relative to /root/reference/pkg/src/lorafuse/.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "af_decode.cuh"
#include "af_forward.cuh"
#include "af_gemv_chain.cuh"
#include "af_llama.cuh"
#include "af_peer.cuh"
#include "af_switch_mma.cuh"
#include "af_switch_umma.cuh"

namespace af {

std::string& last_error_slot() {
    static thread_local std::string slot;
    return slot;
}
int fail(int code, const std::string& msg) {
    last_error_slot() = msg;
    return code;
}
std::atomic<long long> g_launches{0};
// name of the switch kernel the last switch / switch + GEMV call launched (af_last_switch_kernel: bench.py reports it)
static thread_local char g_last_switch_kernel[96] = "none";
static void note_kernel(const char* fmt, int a, int b, int c = -1) {
    if (c >= 0) snprintf(g_last_switch_kernel, sizeof(g_last_switch_kernel), fmt, a, b, c);
    else snprintf(g_last_switch_kernel, sizeof(g_last_switch_kernel), fmt, a, b);
}
// Programmatic dependent launch for the decode GEMV chain (af_set_pdl; env AF_PDL=0 disables).
static std::atomic<int> g_pdl{[] {
    const char* e = getenv("AF_PDL");
    return (e && e[0] == '0') ? 0 : 1;
}()};
// Streaming strategy of the fused decode GEMV (af_set_gemv_variant; env AF_GEMV): 0 = registers
// (LDG.128), 1..4 = shared-memory ring filled by bulk copies (2 KB x1, 2 KB x2, 4 KB x1, 4 KB x2 producers).
static std::atomic<int> g_gemv_variant{[] {
    const char* e = getenv("AF_GEMV");
    return e ? atoi(e) : 0;
}()};
static std::atomic<int> g_gemv_full_sm{[] {
    const char* e = getenv("AF_GEMV_FULL_SM");
    return (e && e[0] == '1') ? 1 : 0;
}()};

// Timeline probe of the fused switch + GEMV launches (af_set_timeline): launch i of the probed
// sequence writes its per-CTA stamps to buffer + i * stride.
static unsigned long long* g_timeline = nullptr;
static int g_timeline_left = 0;
static long long g_timeline_stride = 0;
// tcgen05 / TMEM kernels for eligible tables (af_set_umma; env AF_UMMA=0 turns them off): 1 = tcgen05, 0 = mma.sync
static std::atomic<int> g_umma{[] {
    const char* e = getenv("AF_UMMA");
    return e ? atoi(e) : 1;
}()};
// bf16 pieces of the gated DOWN rows in launches of at most 32 stacked ranks (af_set_umma_pieces; env AF_UMMA_PIECES)
static std::atomic<int> g_umma_pieces{[] {
    const char* e = getenv("AF_UMMA_PIECES");
    return e && atoi(e) == 3 ? 3 : 2;
}()};
static const bool g_force_hilo = [] { const char* e = getenv("AF_FORCE_HILO"); return e && e[0] == '1'; }();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) and occupancy are per DEVICE: what has been configured is
// remembered per device id, so a second GPU in the same process gets its own attribute call.
struct PerDevice {
    int v[64] = {};
    int& cur() {
        int d = 0;
        cudaGetDevice(&d);
        return v[d & 63];
    }
};
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline size_t esize(int dtype) { return dtype == AF_BF16 ? 2 : 4; }

// ---- driver entry point for cuTensorMapEncodeTiled (no link-time libcuda dependency) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

static int make_map(CUtensorMap* out, const void* base, int rows, int cols, long long ld, int box_cols, int box_rows,
                    CUtensorMapSwizzle swz) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return fail(AF_ECUDA, "cuTensorMapEncodeTiled entry point not found");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(AF_ECUDA, "cuTensorMapEncodeTiled failed with code " + std::to_string((int)r));
    return AF_OK;
}

struct DeviceInfo {
    int sm_count = 0, cc_major = 0, cc_minor = 0;
    long long l2 = 0;
    int max_smem_optin = 0;
    bool ok = false;
};
static const DeviceInfo& device_info() {
    static thread_local DeviceInfo info;
    static thread_local int cached_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return info;
    if (info.ok && dev == cached_dev) return info;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return info;
    info.sm_count = prop.multiProcessorCount;
    info.cc_major = prop.major;
    info.cc_minor = prop.minor;
    info.l2 = prop.l2CacheSize;
    info.max_smem_optin = (int)prop.sharedMemPerBlockOptin;
    info.ok = true;
    cached_dev = dev;
    return info;
}

}  // namespace af

using namespace af;

// linalg.py:207-231 `SegmentTable`, device resident.
struct af_table {
    int n_segments = 0;
    int target_dtype = AF_BF16, factor_dtype = AF_BF16;
    std::vector<af_segment_desc> segs;
    SegDev* d_segs = nullptr;
    UnitDev* d_units = nullptr;
    int n_units = 0;
    UnitDev* d_units_umma = nullptr;   // whole-table schedule in 128 x 128 tiles (tcgen05 kernel)
    int n_units_umma = 0;
    CUtensorMap* d_maps = nullptr;  // [5][n_segments]: fma live, fma pristine, mma live, mma pristine, UP bank (swizzled)
    int* d_err = nullptr;
    int* err_word = nullptr;        // where the kernels raise: d_err, or a caller-owned word (af_table_set_error_word)
    Plan* d_plan = nullptr;         // af_plan_build target
    bool fast_fma = false, fast_mma = false, has_pristine = false;
    bool rank16 = true;  // every segment's rank is a multiple of 16
    bool mixed_rank = false;
    bool umma_ok = false;   // tcgen05 path: rank 8 everywhere, every matrix a multiple of 128 x 128
    int max_rank = 0, min_experts = 0;
    long long target_elems = 0;
    int sm_count = 0;
};

// A group of segments that share one input vector (q|k|v, gate|up, or a single matrix) with its
// own work-unit schedule: the fused switch + GEMV launch of one projection of the decode forward.
struct af_group {
    af_table* table = nullptr;
    std::vector<int> segs;
    UnitDev* d_units = nullptr;
    int n_units = 0, grid = 0;
    UnitDev* d_units_umma = nullptr;   // the same phases cut into 128 x 128 tiles (tcgen05 path), when the table allows it
    int n_units_umma = 0, grid_umma = 0;
    int* d_seg_yoff = nullptr;
    int n_phases = 1;
    int x_len[kMaxPhases] = {0, 0, 0, 0}, y_rows[kMaxPhases] = {0, 0, 0, 0};
    long long tiles = 0;
    // tensor-parallel peers (af_group_set_peers): 0 = none
    int n_peers = 0, reduce_mask = 0;
    long long peer_off[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

extern "C" {

int af_abi_version(void) { return AF_ABI_VERSION; }
const char* af_last_error(void) { return last_error_slot().c_str(); }

int af_device_info(int* sm_count, int* cc_major, int* cc_minor, int64_t* l2_bytes) {
    const DeviceInfo& d = device_info();
    if (!d.ok) return fail(AF_ECUDA, "no CUDA device");
    if (sm_count) *sm_count = d.sm_count;
    if (cc_major) *cc_major = d.cc_major;
    if (cc_minor) *cc_minor = d.cc_minor;
    if (l2_bytes) *l2_bytes = d.l2;
    return AF_OK;
}

int64_t af_launch_count(void) { return g_launches.load(); }
const char* af_last_switch_kernel(void) { return g_last_switch_kernel; }

int af_set_pdl(int32_t enable) {
    g_pdl.store(enable ? 1 : 0);
    return AF_OK;
}

int af_set_umma(int32_t enable) {
    g_umma.store(enable ? 1 : 0);
    return AF_OK;
}

int af_set_umma_pieces(int32_t pieces) {
    if (pieces != 2 && pieces != 3) return fail(AF_EVALUE, "the gated DOWN rows split into 2 or 3 bf16 pieces");
    g_umma_pieces.store(pieces);
    return AF_OK;
}

int af_set_gemv_variant(int32_t variant, int32_t full_sm) {
    if (variant < 0 || variant > 4) return fail(AF_EVALUE, "GEMV variant must be 0..4");
    g_gemv_variant.store(variant);
    g_gemv_full_sm.store(full_sm ? 1 : 0);
    return AF_OK;
}

// ------------------------------------------------------------------ table ----

int af_table_destroy(af_table* t) {
    if (!t) return AF_OK;
    if (t->d_segs) cudaFree(t->d_segs);
    if (t->d_units) cudaFree(t->d_units);
    if (t->d_units_umma) cudaFree(t->d_units_umma);
    if (t->d_maps) cudaFree(t->d_maps);
    if (t->d_err) cudaFree(t->d_err);
    if (t->d_plan) cudaFree(t->d_plan);
    delete t;
    return AF_OK;
}

int af_table_create(const af_segment_desc* segments, int32_t n_segments, int32_t target_dtype, int32_t factor_dtype,
                    af_table** out) {
    if (!out) return fail(AF_EVALUE, "out is NULL");
    *out = nullptr;
    // ---- validation first, nothing touched (linalg.py:219-228, 199-205) ----
    if (n_segments < 1 || !segments) return fail(AF_EDIM, "segment table is empty");
    if ((target_dtype != AF_BF16 && target_dtype != AF_F32) || (factor_dtype != AF_BF16 && factor_dtype != AF_F32))
        return fail(AF_EPRECISION, "unknown precision tag");
    const size_t te = esize(target_dtype);
    for (int i = 0; i < n_segments; ++i) {
        const af_segment_desc& s = segments[i];
        if (s.d_out < 0 || s.d_in < 0 || s.rank < 0 || s.n_experts < 1)
            return fail(AF_EDIM, "segment " + std::to_string(i) + ": negative extent or empty bank");
        if (s.d_out > 0 && s.d_in > 0 && !s.target) return fail(AF_EDIM, "segment " + std::to_string(i) + ": target is NULL");
        if (s.ld_target < s.d_in) return fail(AF_EDIM, "segment " + std::to_string(i) + ": target pitch below d_in");
        if (s.rank > 0 && (s.ld_down < s.d_in || s.ld_up < s.rank))
            return fail(AF_EDIM, "segment " + std::to_string(i) + ": factor pitch below its row length");
        if (s.rank > 0 && s.d_out > 0 && s.d_in > 0 && (!s.down || !s.up))
            return fail(AF_EDIM, "segment " + std::to_string(i) + ": factor pointer is NULL");
    }
    {  // distinct, non-overlapping targets (linalg.py:222-228 keyed on identity; here on address ranges)
        struct Range {
            uintptr_t lo, hi;
            int idx;
        };
        std::vector<Range> rs;
        for (int i = 0; i < n_segments; ++i) {
            const af_segment_desc& s = segments[i];
            if (s.d_out == 0 || s.d_in == 0) continue;
            const uintptr_t lo = reinterpret_cast<uintptr_t>(s.target);
            const uintptr_t hi = lo + ((uintptr_t)(s.d_out - 1) * (uintptr_t)s.ld_target + (uintptr_t)s.d_in) * te;
            rs.push_back({lo, hi, i});
        }
        std::sort(rs.begin(), rs.end(), [](const Range& a, const Range& b) { return a.lo < b.lo; });
        for (size_t i = 1; i < rs.size(); ++i)
            if (rs[i].lo < rs[i - 1].hi)
                return fail(AF_EALIAS, "segments " + std::to_string(rs[i - 1].idx) + " and " + std::to_string(rs[i].idx) +
                                           " share one target matrix");
    }
    const DeviceInfo& dinfo = device_info();
    if (!dinfo.ok) return fail(AF_ECUDA, "no CUDA device");

    af_table* t = new af_table();
    t->n_segments = n_segments;
    t->target_dtype = target_dtype;
    t->factor_dtype = factor_dtype;
    t->segs.assign(segments, segments + n_segments);
    t->sm_count = dinfo.sm_count;
    t->has_pristine = true;
    t->min_experts = segments[0].n_experts;
    bool fma_ok = (target_dtype == AF_BF16), mma_ok = (target_dtype == AF_BF16 && factor_dtype == AF_BF16);
    std::vector<SegDev> hs(n_segments);
    long long total_tiles = 0;
    for (int i = 0; i < n_segments; ++i) {
        const af_segment_desc& s = segments[i];
        SegDev& d = hs[i];
        d.target = s.target;
        d.pristine = s.pristine;
        d.down = s.down;
        d.up = s.up;
        d.d_out = s.d_out;
        d.d_in = s.d_in;
        d.rank = s.rank;
        d.n_experts = s.n_experts;
        d.ld_target = s.ld_target;
        d.ld_down = s.ld_down;
        d.ld_up = s.ld_up;
        d.down_estride = s.down_expert_stride;
        d.up_estride = s.up_expert_stride;
        if (!s.pristine) t->has_pristine = false;
        t->max_rank = std::max(t->max_rank, s.rank);
        t->min_experts = std::min(t->min_experts, s.n_experts);
        t->target_elems += (long long)s.d_out * s.d_in;
        total_tiles += (long long)((s.d_out + kTM - 1) / kTM) * ((s.d_in + kTN - 1) / kTN);
        // TMA: 16-byte aligned base and row pitch
        const bool tma_ok = s.d_out > 0 && s.d_in > 0 && (reinterpret_cast<uintptr_t>(s.target) % 16 == 0) &&
                            (s.ld_target % 8 == 0) &&
                            (!s.pristine || reinterpret_cast<uintptr_t>(s.pristine) % 16 == 0);
        if (!tma_ok) fma_ok = mma_ok = false;
        // tensor path: dense UP rows (ld_up == rank), rank a multiple of 8, 16-byte aligned factor blocks
        const bool fac_ok = s.rank > 0 && s.rank % 8 == 0 && s.ld_up == s.rank && (s.up_expert_stride % 8 == 0) &&
                            (reinterpret_cast<uintptr_t>(s.up) % 16 == 0) && (s.ld_down % 8 == 0) &&
                            (s.down_expert_stride % 8 == 0) && (reinterpret_cast<uintptr_t>(s.down) % 16 == 0);
        if (!fac_ok) mma_ok = false;
        // ranks fetched through the swizzled UP map need the bank packed as one [N * d_out][rank] matrix
        if (up_swizzled(s.rank) && s.up_expert_stride != (long long)s.d_out * s.rank) mma_ok = false;
        if (s.rank % 16 != 0) t->rank16 = false;
        if (s.rank != segments[0].rank) t->mixed_rank = true;
    }
    t->fast_fma = fma_ok;
    t->fast_mma = mma_ok;
    t->umma_ok = mma_ok;
    for (int i = 0; i < n_segments; ++i) {
        const af_segment_desc& s = segments[i];
        const bool rank_ok = s.rank == segments[0].rank && (s.rank == 8 || s.rank == 16 || s.rank == 32 || s.rank == 64);
        // Any matrix of at least one 128 x 128 tile: ragged edges (tensor-parallel shards: ffn / tp = 2752, 1376, 1728 ...)
        // are partial tiles -- TMA zero-fills what it loads out of bounds and clips what it stores, the UP copy
        // of a partial row tile is cut at d_out, slab and input-vector columns past d_in are zeros.
        if (!rank_ok || s.d_out < kUM || s.d_in < kUN) t->umma_ok = false;
    }

    // ---- work units: column strips of kTN columns cut into runs of row tiles ----
    // Static round-robin schedule over the persistent grid: aim for ~32 units per SM so the
    // tail imbalance stays below ~3 %, but keep runs long enough to amortise the slab staging.
    long long per_unit = total_tiles / ((long long)std::max(1, t->sm_count) * 32);
    per_unit = std::max(1LL, std::min(64LL, per_unit));
    std::vector<UnitDev> units;
    for (int i = 0; i < n_segments; ++i) {
        const af_segment_desc& s = segments[i];
        if (s.d_out == 0 || s.d_in == 0) continue;
        const int rows_per_unit = (int)per_unit * kTM;
        for (int c0 = 0; c0 < s.d_in; c0 += kTN)
            for (int r0 = 0; r0 < s.d_out; r0 += rows_per_unit)
                units.push_back({i, r0, std::min(rows_per_unit, s.d_out - r0), c0});
    }
    // Largest units first: with the round-robin walk (unit u -> CTA u % grid) every CTA then gets the
    // same mix of sizes.  Unsorted, segments of different shapes alias with the grid size (42 % more
    // work on the busiest SM for Llama-2-13B shapes, 10 % for Llama-3-8B); sorted, < 1 %.
    std::stable_sort(units.begin(), units.end(), [&](const UnitDev& a, const UnitDev& b) {
        const long long wa = (long long)a.rows * std::min(kTN, segments[a.seg].d_in - a.col0);
        const long long wb = (long long)b.rows * std::min(kTN, segments[b.seg].d_in - b.col0);
        return wa > wb;
    });
    t->n_units = (int)units.size();
    // the same walk in 128 x 128 tiles for the tcgen05 kernel
    std::vector<UnitDev> units_u;
    if (t->umma_ok) {
        long long tiles_u = 0;
        for (int i = 0; i < n_segments; ++i)
            tiles_u += (long long)((segments[i].d_out + kUM - 1) / kUM) * ((segments[i].d_in + kUN - 1) / kUN);
        long long per_u = std::max(1LL, std::min(32LL, tiles_u / ((long long)std::max(1, t->sm_count) * 32)));
        for (int i = 0; i < n_segments; ++i) {
            const af_segment_desc& s = segments[i];
            const int rows_per_unit = (int)per_u * kUM;
            for (int c0 = 0; c0 < s.d_in; c0 += kUN)
                for (int r0 = 0; r0 < s.d_out; r0 += rows_per_unit)
                    units_u.push_back({i, r0, std::min(rows_per_unit, s.d_out - r0), c0, 0, 0});
        }
        std::stable_sort(units_u.begin(), units_u.end(), [&](const UnitDev& a, const UnitDev& b) { return a.rows > b.rows; });
        t->n_units_umma = (int)units_u.size();
    }

    cudaError_t e = cudaMalloc(&t->d_segs, sizeof(SegDev) * n_segments);
    if (e == cudaSuccess) e = cudaMemcpy(t->d_segs, hs.data(), sizeof(SegDev) * n_segments, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && t->n_units) e = cudaMalloc(&t->d_units, sizeof(UnitDev) * units.size());
    if (e == cudaSuccess && t->n_units)
        e = cudaMemcpy(t->d_units, units.data(), sizeof(UnitDev) * units.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && t->n_units_umma) e = cudaMalloc(&t->d_units_umma, sizeof(UnitDev) * units_u.size());
    if (e == cudaSuccess && t->n_units_umma)
        e = cudaMemcpy(t->d_units_umma, units_u.data(), sizeof(UnitDev) * units_u.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&t->d_err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(t->d_err, 0, sizeof(int));
    t->err_word = t->d_err;
    if (e == cudaSuccess) e = cudaMalloc(&t->d_plan, sizeof(Plan));
    if (e == cudaSuccess) e = cudaMemset(t->d_plan, 0, sizeof(Plan));
    if (e != cudaSuccess) {
        af_table_destroy(t);
        return fail(AF_ECUDA, std::string("table upload: ") + cudaGetErrorString(e));
    }
    if (t->fast_fma) {
        // [5], [6]: 128 x 64 boxes of the tcgen05 path (live, pristine); [7]: its UP blocks (128 rows x rank, swizzled)
        std::vector<CUtensorMap> maps((size_t)8 * n_segments);
        std::memset(maps.data(), 0, sizeof(CUtensorMap) * maps.size());
        for (int i = 0; i < n_segments; ++i) {
            const af_segment_desc& s = segments[i];
            const void* pr = s.pristine ? s.pristine : s.target;
            int rc = make_map(&maps[0 * n_segments + i], s.target, s.d_out, s.d_in, s.ld_target, kTN, kTM, CU_TENSOR_MAP_SWIZZLE_NONE);
            if (!rc) rc = make_map(&maps[1 * n_segments + i], pr, s.d_out, s.d_in, s.ld_target, kTN, kTM, CU_TENSOR_MAP_SWIZZLE_NONE);
            if (!rc) rc = make_map(&maps[2 * n_segments + i], s.target, s.d_out, s.d_in, s.ld_target, kBoxCols, kMR, CU_TENSOR_MAP_SWIZZLE_128B);
            if (!rc) rc = make_map(&maps[3 * n_segments + i], pr, s.d_out, s.d_in, s.ld_target, kBoxCols, kMR, CU_TENSOR_MAP_SWIZZLE_128B);
            if (!rc && t->fast_mma && up_swizzled(s.rank)) {
                // UP bank of the segment as one [N * d_out][rank] matrix; swizzle span = row bytes
                const CUtensorMapSwizzle sw = s.rank == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                              : s.rank == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
                rc = make_map(&maps[4 * n_segments + i], s.up, s.n_experts * s.d_out, s.rank, s.rank, s.rank, kMR, sw);
            }
            if (!rc && t->umma_ok) {
                rc = make_map(&maps[5 * n_segments + i], s.target, s.d_out, s.d_in, s.ld_target, kUBoxCols, kUM, CU_TENSOR_MAP_SWIZZLE_128B);
                if (!rc) rc = make_map(&maps[6 * n_segments + i], pr, s.d_out, s.d_in, s.ld_target, kUBoxCols, kUM, CU_TENSOR_MAP_SWIZZLE_128B);
                if (!rc && s.rank > 8) {
                    const CUtensorMapSwizzle sw = s.rank == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : s.rank == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
                    rc = make_map(&maps[7 * n_segments + i], s.up, s.n_experts * s.d_out, s.rank, s.rank, s.rank, kUM, sw);
                }
            }
            if (rc) {
                af_table_destroy(t);
                return rc;
            }
        }
        e = cudaMalloc(&t->d_maps, sizeof(CUtensorMap) * maps.size());
        if (e == cudaSuccess) e = cudaMemcpy(t->d_maps, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            af_table_destroy(t);
            return fail(AF_ECUDA, std::string("tensor map upload: ") + cudaGetErrorString(e));
        }
    }
    *out = t;
    return AF_OK;
}

int af_table_info(const af_table* t, int32_t* n_segments, int64_t* target_elems, int32_t* n_units, int32_t* fast_path) {
    if (!t) return fail(AF_EVALUE, "table is NULL");
    if (n_segments) *n_segments = t->n_segments;
    if (target_elems) *target_elems = t->target_elems;
    if (n_units) *n_units = t->n_units;
    if (fast_path) *fast_path = (t->fast_fma ? 1 : 0) | (t->fast_mma ? 2 : 0) | ((t->umma_ok && g_umma.load()) ? 4 : 0);
    return AF_OK;
}

const char* af_flag_message(int32_t flag) {
    switch (flag) {
        case AF_OK: return "ok";
        case AF_EINDEX: return "a device decision names an expert outside the bank";
        case AF_EVALUE: return "a device decision carries more experts than max_k";
        case AF_ESTATE: return "the KV cache is full (position >= max_seq)";
        case AF_ECUDA: return "a chained launch timed out at a phase barrier (a CTA of the launch was not co-resident)";
        default: return "a kernel raised an unknown status";
    }
}

int af_table_set_error_word(af_table* t, int32_t* word_dev) {
    if (!t) return fail(AF_EVALUE, "table is NULL");
    t->err_word = word_dev ? word_dev : t->d_err;
    return AF_OK;
}

int af_table_status(af_table* t, void* stream) {
    if (!t) return fail(AF_EVALUE, "table is NULL");
    int flag = 0;
    AF_CUDA_TRY(cudaMemcpyAsync(&flag, t->err_word, sizeof(int), cudaMemcpyDeviceToHost, as_stream(stream)));
    AF_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
    if (flag) {
        AF_CUDA_TRY(cudaMemsetAsync(t->err_word, 0, sizeof(int), as_stream(stream)));
        return fail(flag, af_flag_message(flag));
    }
    return AF_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ switch launch ----

namespace af {

template <int KS, bool BA, bool GEMV = false, bool TL = false>
static int launch_mma(const MmaParams& mp, int grid, cudaStream_t st) {
    using L = MmaLayout<KS, BA, GEMV>;
    static PerDevice configured;
    if (!configured.cur()) {
        AF_CUDA_TRY(cudaFuncSetAttribute(switch_mma_kernel<KS, BA, GEMV, TL>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::total));
        configured.cur() = 1;
    }
    MmaParams mp2 = mp;
    static const int env_stages = [] { const char* e = getenv("AF_MMA_STAGES"); return e ? atoi(e) : 0; }();
    static const int env_depth = [] { const char* e = getenv("AF_STORE_DEPTH"); return e ? atoi(e) : -1; }();
    mp2.n_stages = std::min(L::stages, kMmaDefaultStages);
    (void)env_stages;
    mp2.store_depth = (env_depth >= 0 && env_depth <= 3) ? env_depth : kStoreDepth;
    static const int env_upsw = [] { const char* e = getenv("AF_UP_SWIZZLE"); return (e && e[0] == '0') ? 0 : 1; }();
    mp2.up_swizzle_ok = env_upsw;
    static const int env_dbg2 = [] { const char* e = getenv("AF_DBG"); return e ? atoi(e) : 0; }();
    mp2.dbg = env_dbg2 ^ 24;  // bits 8 / 16: L2 evict-first hint on the W loads / stores, on unless AF_DBG flips them
    if (mp2.store_depth > mp2.n_stages - 2) mp2.store_depth = mp2.n_stages - 2;
    if constexpr (GEMV) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kMmaThreadsGemv);
        cfg.dynamicSmemBytes = L::total;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = mp2.pdl ? 1 : 0;
        AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, switch_mma_kernel<KS, BA, GEMV, TL>, mp2));
    } else {
        switch_mma_kernel<KS, BA, GEMV, TL><<<grid, kMmaThreads, L::total, st>>>(mp2);
    }
    AF_LAUNCH_CHECK("switch_mma_kernel");
    note_kernel("switch_mma_kernel<KS=%d,BA=%d,GEMV=%d> (mma.sync)", KS, (int)BA, (int)GEMV);
    return AF_OK;
}

// Stacked ranks (2 k r in the steady switch) up to which the tcgen05 kernel is used: 256, K-chunked above 32
// (af_switch_umma.cuh), for tables of rank 8 / 16 / 32; rank 64 up to 64.  AF_UMMA_MAX_RANKS[_CHAIN] override (A/B runs).
static const int kUmmaMaxRanks = [] { const char* e = getenv("AF_UMMA_MAX_RANKS"); return e ? atoi(e) : 256; }();
static const int kUmmaMaxRanksChain = [] { const char* e = getenv("AF_UMMA_MAX_RANKS_CHAIN"); return e ? atoi(e) : 256; }();
// 1: launches of 33..64 stacked ranks stream the UP operand in 32-rank chunks too (same shared memory, twice the
// barrier traffic: measured 1.5 % slower on Llama-3-8B shapes, so off)
static const int kUmmaChunk64 = [] { const char* e = getenv("AF_UMMA_CHUNK64"); return e ? atoi(e) : 0; }();
// tcgen05 / TMEM kernel (af_switch_umma.cuh).  NB = k-groups of 8 stacked ranks per half, CH = k-groups per UP stage.
template <int NB, bool GEMV, int CH, int PC, bool PEERS>
static int launch_umma_k(const MmaParams& mp, int grid, cudaStream_t st) {
    using L = UmmaLayout<NB, GEMV, CH, PC>;
    static PerDevice configured;
    if (!configured.cur()) {
        AF_CUDA_TRY(cudaFuncSetAttribute(switch_umma_kernel<NB, GEMV, CH, PC, PEERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::total));
        configured.cur() = 1;
    }
    if (mp.n_phases > 1) {
        // The phases of a chained launch meet at in-kernel grid barriers: every CTA must be resident at once.  One CTA
        // per SM by construction; refuse the launch when the device cannot hold it (a smaller partition, MIG) instead
        // of running into the barrier timeout.
        static PerDevice occ_checked;
        if (!occ_checked.cur()) {
            int per_sm = 0;
            AF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, switch_umma_kernel<NB, GEMV, CH, PC, PEERS>, kUThreads, L::total));
            const DeviceInfo& di = device_info();
            if (per_sm < 1 || grid > di.sm_count * per_sm)
                return fail(AF_ESTATE, "a chained launch needs all its CTAs co-resident: " + std::to_string(grid) + " CTAs, device holds " +
                                           std::to_string(di.sm_count * per_sm));
            occ_checked.cur() = 1;
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kUThreads);
    cfg.dynamicSmemBytes = L::total;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = mp.pdl ? 1 : 0;
    AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, switch_umma_kernel<NB, GEMV, CH, PC, PEERS>, mp));
    AF_LAUNCH_CHECK("switch_umma_kernel");
    note_kernel(PC == 3 ? "switch_umma_kernel<NB=%d,GEMV=%d,CH=%d,PC=3> (tcgen05 + TMEM)"
                        : (PEERS ? "switch_umma_kernel<NB=%d,GEMV=%d,CH=%d,PEERS> (tcgen05 + TMEM)" : "switch_umma_kernel<NB=%d,GEMV=%d,CH=%d> (tcgen05 + TMEM)"),
                NB, (int)GEMV, CH);
    return AF_OK;
}

template <int NB, bool GEMV, int CH = NB, int PC = 2>
static int launch_umma(const MmaParams& mp, int grid, cudaStream_t st) {
    // tensor-parallel pushes (af_group_set_peers) are a separate instantiation of the GEMV kernels
    if (GEMV && mp.n_peers > 0) return launch_umma_k<NB, GEMV, CH, PC, GEMV>(mp, grid, st);
    return launch_umma_k<NB, GEMV, CH, PC, false>(mp, grid, st);
}

// Largest stacked rank ONE tcgen05 launch over this table takes (0: the table is not eligible at all)
static int umma_rank_limit(const af_table* t) {
    if (!t->umma_ok || !g_umma.load()) return 0;
    return t->max_rank <= 32 ? 256 : 64;
}
template <bool GEMV>
static int dispatch_umma(const af_table* t, int s_bound, const MmaParams& mp, int grid, cudaStream_t st) {
    // up to 32 stacked ranks: the gated DOWN rows in two or three bf16 pieces (af_set_umma_pieces; see UmmaLayout)
    if (s_bound <= 32) return g_umma_pieces.load() == 3 ? launch_umma<4, GEMV, 4, 3>(mp, grid, st) : launch_umma<4, GEMV>(mp, grid, st);
    if (s_bound <= 64) return (kUmmaChunk64 && t->max_rank <= 32) ? launch_umma<8, GEMV, 4>(mp, grid, st) : launch_umma<8, GEMV>(mp, grid, st);
    // 128 stacked ranks: UP chunks of 64 ranks (three 16 KB stages) beat chunks of 32 (six 8 KB stages) -- half the chunk
    // barriers per tile: 2.41 against 2.61 ms on 24 layers of a Llama-2-70B tp8 shard, 13.0 against 14.5 ms per shard step
    static const int ch128 = [] { const char* e = getenv("AF_UMMA_CH128"); return e ? atoi(e) : 8; }();
    if (s_bound <= 128) return ch128 == 8 ? launch_umma<16, GEMV, 8>(mp, grid, st) : launch_umma<16, GEMV, 4>(mp, grid, st);
    return launch_umma<32, GEMV, 4>(mp, grid, st);
}

template <typename FT, bool EXACT, bool F2>
static int launch_tma(const SwitchParams& p, int grid, cudaStream_t st) {
    static PerDevice configured;
    const int smem = (int)sizeof(SwitchSmem) + 128;
    if (!configured.cur()) {
        AF_CUDA_TRY(cudaFuncSetAttribute(switch_tma_kernel<FT, EXACT, F2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        configured.cur() = 1;
    }
    switch_tma_kernel<FT, EXACT, F2><<<grid, kConsumers + 32, smem, st>>>(p);
    AF_LAUNCH_CHECK("switch_tma_kernel");
    note_kernel("switch_tma_kernel<EXACT=%d,F2=%d> (CUDA cores)", (int)EXACT, (int)F2);
    return AF_OK;
}

template <bool EXACT>
static int launch_any(const af_table* t, const SwitchParams& p, int grid, cudaStream_t st) {
    if (t->target_dtype == AF_BF16 && t->factor_dtype == AF_BF16)
        switch_any_kernel<__nv_bfloat16, __nv_bfloat16, EXACT><<<grid, kTN, 0, st>>>(p);
    else if (t->target_dtype == AF_BF16)
        switch_any_kernel<__nv_bfloat16, float, EXACT><<<grid, kTN, 0, st>>>(p);
    else if (t->factor_dtype == AF_BF16)
        switch_any_kernel<float, __nv_bfloat16, EXACT><<<grid, kTN, 0, st>>>(p);
    else
        switch_any_kernel<float, float, EXACT><<<grid, kTN, 0, st>>>(p);
    AF_LAUNCH_CHECK("switch_any_kernel");
    return AF_OK;
}

static int check_host_decision(const af_table* t, const af_decision* d, const char* which) {
    if (!d) return AF_OK;
    if (d->k < 0 || d->k > AF_MAX_K) return fail(AF_EVALUE, std::string(which) + " decision: k outside [0, AF_MAX_K]");
    for (int j = 0; j < d->k; ++j)
        if (d->ids[j] < 0 || d->ids[j] >= t->min_experts)
            return fail(AF_EINDEX, std::string(which) + " decision: expert id " + std::to_string(d->ids[j]) +
                                       " outside bank of " + std::to_string(t->min_experts));
    return AF_OK;
}

// Common launcher.  host_plan_override != nullptr: af_sgmm (materialised segments).
static int run_switch(af_table* t, const af_decision* prev_dev, const af_decision* cur_dev, const af_decision* prev_host,
                      const af_decision* cur_host, int max_k, float scale, int mode, int compute,
                      const Plan* host_plan_override, cudaStream_t st) {
    if (!t) return fail(AF_EVALUE, "table is NULL");
    if (mode != AF_SWITCH_INPLACE && mode != AF_SWITCH_FROM_PRISTINE) return fail(AF_EVALUE, "unknown switch mode");
    if (compute < AF_COMPUTE_AUTO || compute > AF_COMPUTE_MMA) return fail(AF_EVALUE, "unknown compute mode");
    if (mode == AF_SWITCH_FROM_PRISTINE && !t->has_pristine)
        return fail(AF_ESTATE, "FROM_PRISTINE needs a pristine copy of every segment");
    const bool use_dev = (prev_dev || cur_dev) && !host_plan_override;
    if (use_dev && ((prev_host && !prev_dev) || (cur_host && !cur_dev)))
        return fail(AF_EVALUE, "decisions must be all device-resident or all host-resident");
    if (use_dev && (max_k < 1 || max_k > AF_MAX_K)) return fail(AF_EVALUE, "max_k outside [1, AF_MAX_K]");
    const bool exact = compute == AF_COMPUTE_EXACT;

    SwitchParams p{};
    p.segs = t->d_segs;
    p.units = t->d_units;
    p.n_units = t->n_units;
    p.from_pristine = mode == AF_SWITCH_FROM_PRISTINE;
    p.prev_dev = prev_dev;
    p.cur_dev = cur_dev;
    p.use_dev = use_dev ? 1 : 0;
    p.scale = scale;
    p.n_experts_limit = t->min_experts;
    p.err_flag = t->err_word;
    int n_blocks_bound;
    if (host_plan_override) {
        p.host_plan = *host_plan_override;
        n_blocks_bound = p.host_plan.n_blocks;
    } else if (!use_dev) {
        int rc = check_host_decision(t, prev_host, "previous");
        if (!rc) rc = check_host_decision(t, cur_host, "current");
        if (rc) return rc;
        build_plan(p.host_plan, p.from_pristine ? nullptr : prev_host, cur_host, scale, exact, t->min_experts);
        n_blocks_bound = p.host_plan.n_blocks;
        if (n_blocks_bound == 0 && !p.from_pristine) return AF_OK;  // nothing changes: no launch
    } else {
        n_blocks_bound = (p.from_pristine || !prev_dev ? 0 : max_k) + (cur_dev ? max_k : 0);
    }
    p.max_blocks = std::min(n_blocks_bound, kMaxBlocks);
    if (t->n_units == 0) return AF_OK;
    const int s_bound = n_blocks_bound * t->max_rank;

    const bool want_mma = compute == AF_COMPUTE_MMA || compute == AF_COMPUTE_AUTO;
    const bool umma_fits = t->fast_mma && t->n_units_umma && !host_plan_override && s_bound <= std::min(kUmmaMaxRanks, umma_rank_limit(t));
    const bool mma_fits = t->fast_mma && s_bound <= kMmaMaxKS * 16;
    if (compute == AF_COMPUTE_MMA && !mma_fits && !umma_fits)
        return fail(AF_EVALUE, "tensor path needs bf16 targets and factors, rank % 8 == 0, 16-byte aligned rows and at most 64 stacked "
                               "ranks (256 on the tcgen05 path: one rank of 8 / 16 / 32 per table, matrices multiples of 128)");
    const int S = t->n_segments;
    if (want_mma && umma_fits) {
        MmaParams mp{};
        mp.base = p;
        mp.base.units = t->d_units_umma;
        mp.base.n_units = t->n_units_umma;
        mp.tmaps_ld = t->d_maps + (size_t)(p.from_pristine ? 6 : 5) * S;
        mp.tmaps_st = t->d_maps + (size_t)5 * S;
        mp.tmaps_up = t->d_maps + (size_t)7 * S;
        mp.n_chain_segs = 0;
        mp.n_phases = 1;
        const int grid = std::min(t->n_units_umma, t->sm_count);
        static const int env_dbg3 = [] { const char* e = getenv("AF_DBG"); return e ? atoi(e) : 0; }();
        mp.dbg = env_dbg3 ^ 24;
        return dispatch_umma<false>(t, s_bound, mp, grid, st);
    }
    if (want_mma && mma_fits) {
        MmaParams mp{};
        mp.base = p;
        mp.tmaps_ld = t->d_maps + (size_t)(p.from_pristine ? 3 : 2) * S;
        mp.tmaps_st = t->d_maps + (size_t)2 * S;
        mp.tmaps_up = t->d_maps + (size_t)4 * S;
        mp.mixed_rank = t->mixed_rank ? 1 : 0;
        const int grid = std::min(t->n_units, t->sm_count);
        const int ks = std::max(1, (s_bound + 15) / 16);
        // block-accumulate form when every block is a whole number of rank-16 steps and the hi/lo
        // form would need more than two steps (it doubles the tensor work)
        const bool ba = t->rank16 && ks > 2 && !g_force_hilo;
        switch (ks) {
            case 1: return launch_mma<1, false>(mp, grid, st);
            case 2: return launch_mma<2, false>(mp, grid, st);
            case 3: return ba ? launch_mma<3, true>(mp, grid, st) : launch_mma<3, false>(mp, grid, st);
            default: return ba ? launch_mma<4, true>(mp, grid, st) : launch_mma<4, false>(mp, grid, st);
        }
    }
    if (t->fast_fma) {
        p.tmaps_src = t->d_maps + (size_t)(p.from_pristine ? 1 : 0) * S;
        p.tmaps_dst = t->d_maps;
        const int grid = std::min(t->n_units, t->sm_count);
        if (t->factor_dtype == AF_BF16)
            return exact ? launch_tma<__nv_bfloat16, true, false>(p, grid, st) : launch_tma<__nv_bfloat16, false, true>(p, grid, st);
        return exact ? launch_tma<float, true, false>(p, grid, st) : launch_tma<float, false, true>(p, grid, st);
    }
    const int grid = std::min(t->n_units, t->sm_count * 8);
    return exact ? launch_any<true>(t, p, grid, st) : launch_any<false>(t, p, grid, st);
}

}  // namespace af

extern "C" {

int af_fused_switch(af_table* table, const af_decision* prev_dev, const af_decision* cur_dev, const af_decision* prev_host,
                    const af_decision* cur_host, int32_t max_k, float scale, int32_t mode, int32_t compute, void* stream) {
    return run_switch(table, prev_dev, cur_dev, prev_host, cur_host, max_k, scale, mode, compute, nullptr, as_stream(stream));
}

int af_merge(af_table* table, const af_decision* dec_dev, const af_decision* dec_host, int32_t max_k, float scale,
             int32_t compute, void* stream) {
    return run_switch(table, nullptr, dec_dev, nullptr, dec_host, max_k, scale, AF_SWITCH_INPLACE, compute, nullptr,
                      as_stream(stream));
}

int af_unmerge(af_table* table, const af_decision* dec_dev, const af_decision* dec_host, int32_t max_k, float scale,
               int32_t compute, void* stream) {
    return run_switch(table, dec_dev, nullptr, dec_host, nullptr, max_k, scale, AF_SWITCH_INPLACE, compute, nullptr,
                      as_stream(stream));
}

int af_sgmm(af_table* table, int32_t sign, int32_t compute, void* stream) {
    if (sign != 1 && sign != -1) return fail(AF_EVALUE, "sign must be +1 or -1");  // linalg.py:323-324
    if (!table) return fail(AF_EVALUE, "table is NULL");
    Plan plan{};
    plan.n_blocks = 1;
    plan.expert[0] = 0;
    if (compute == AF_COMPUTE_EXACT) {
        plan.weight[0] = 1.0f;            // 1 * down is exact; the sign is applied as `block -= outer`
        plan.negate[0] = sign < 0 ? 1 : 0;
    } else {
        plan.weight[0] = (float)sign;
        plan.negate[0] = 0;
    }
    return run_switch(table, nullptr, nullptr, nullptr, nullptr, 1, 1.0f, AF_SWITCH_INPLACE, compute, &plan, as_stream(stream));
}

int af_refresh_from_pristine(af_table* t, void* stream) {
    if (!t) return fail(AF_EVALUE, "table is NULL");
    if (!t->has_pristine) return fail(AF_ESTATE, "no pristine copy registered");
    const size_t es = esize(t->target_dtype);
    for (const af_segment_desc& s : t->segs) {
        if (s.d_out == 0 || s.d_in == 0) continue;
        AF_CUDA_TRY(cudaMemcpy2DAsync(s.target, s.ld_target * es, s.pristine, s.ld_target * es, (size_t)s.d_in * es,
                                      s.d_out, cudaMemcpyDeviceToDevice, as_stream(stream)));
    }
    return AF_OK;
}

int af_max_deviation(af_table* t, float* out_dev, void* stream) {
    if (!t || !out_dev) return fail(AF_EVALUE, "NULL argument");
    if (!t->has_pristine) return fail(AF_ESTATE, "no pristine copy registered");
    cudaStream_t st = as_stream(stream);
    AF_CUDA_TRY(cudaMemsetAsync(out_dev, 0, sizeof(float), st));
    for (const af_segment_desc& s : t->segs) {
        if (s.d_out == 0 || s.d_in == 0) continue;
        const long long n = (long long)s.d_out * s.d_in;
        const int grid = (int)std::min<long long>((n + 1023) / 1024, (long long)t->sm_count * 8);
        if (t->target_dtype == AF_BF16)
            max_dev_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(s.target),
                                                               reinterpret_cast<const __nv_bfloat16*>(s.pristine), s.d_out,
                                                               s.d_in, s.ld_target, reinterpret_cast<unsigned*>(out_dev));
        else
            max_dev_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(s.target),
                                                       reinterpret_cast<const float*>(s.pristine), s.d_out, s.d_in,
                                                       s.ld_target, reinterpret_cast<unsigned*>(out_dev));
        AF_LAUNCH_CHECK("max_dev_kernel");
    }
    return AF_OK;
}

// ------------------------------------------------------------------ fused switch + GEMV ----

int af_group_destroy(af_group* g) {
    if (!g) return AF_OK;
    if (g->d_units) cudaFree(g->d_units);
    if (g->d_units_umma) cudaFree(g->d_units_umma);
    if (g->d_seg_yoff) cudaFree(g->d_seg_yoff);
    delete g;
    return AF_OK;
}

int af_chain_create(af_table* t, const int32_t* seg_ids, const int32_t* phase_len, int32_t n_phases, af_group** out) {
    return af_chain_create_weighted(t, seg_ids, phase_len, n_phases, nullptr, 0, out);
}

int af_chain_create_weighted(af_table* t, const int32_t* seg_ids, const int32_t* phase_len, int32_t n_phases, const float* cta_share,
                             int32_t n_cta, af_group** out) {
    if (!out) return fail(AF_EVALUE, "out is NULL");
    if (cta_share && n_cta < 1) return fail(AF_EVALUE, "cta_share needs n_cta >= 1");
    if (cta_share)
        for (int i = 0; i < n_phases * n_cta; ++i)
            if (!(cta_share[i] > 0.0f) || !std::isfinite(cta_share[i])) return fail(AF_EVALUE, "cta_share entries must be positive and finite");
    *out = nullptr;
    if (!t || !seg_ids || !phase_len || n_phases < 1) return fail(AF_EDIM, "segment group is empty");
    if (n_phases > kMaxPhases) return fail(AF_EVALUE, "a chain holds at most 4 phases");
    {
        int total_segs = 0;
        for (int ph = 0; ph < n_phases; ++ph) total_segs += phase_len[ph] > 0 ? phase_len[ph] : 0;
        if (total_segs > kSegCache) return fail(AF_EVALUE, "a chain holds at most 12 segments");
    }
    if (!t->fast_mma)
        return fail(AF_EPRECISION, "the fused switch + GEMV needs the tensor path: bf16 targets and factors, rank % 8 == 0, "
                                   "16-byte aligned rows");
    std::vector<int> yoff(t->n_segments, 0);
    std::vector<char> seen(t->n_segments, 0);
    af_group* g = new af_group();
    g->table = t;
    g->n_phases = n_phases;
    int n = 0;
    for (int ph = 0; ph < n_phases; ++ph) {
        if (phase_len[ph] < 1) { delete g; return fail(AF_EDIM, "segment group is empty"); }
        int x_len = -1, rows = 0;
        for (int i = 0; i < phase_len[ph]; ++i) {
            const int sidx = seg_ids[n + i];
            int rc = AF_OK;
            if (sidx < 0 || sidx >= t->n_segments) rc = fail(AF_EINDEX, "segment id outside the table");
            else if (seen[sidx]) rc = fail(AF_EALIAS, "segment listed twice in one group");
            else if (t->segs[sidx].d_out < 1 || t->segs[sidx].d_in < 1) rc = fail(AF_EDIM, "empty segment in a GEMV group");
            else if (x_len >= 0 && t->segs[sidx].d_in != x_len)
                rc = fail(AF_EDIM, "segments of one group must share d_in (one input vector)");
            if (rc) { delete g; return rc; }
            seen[sidx] = 1;
            x_len = t->segs[sidx].d_in;
            yoff[sidx] = rows;
            rows += t->segs[sidx].d_out;
        }
        g->x_len[ph] = x_len;
        g->y_rows[ph] = rows;
        n += phase_len[ph];
    }
    g->segs.assign(seg_ids, seg_ids + n);
    // ---- schedule: per phase, the tiles in (segment, column strip, row tile) order cut into one
    //      contiguous span per CTA -- every SM streams the same number of tiles (+-1) and restages
    //      the DOWN slab only when its span crosses into another strip.  A CTA's spans of all phases
    //      are concatenated into its unit list.  Built for a tile geometry: 32 x 256 (mma.sync kernel)
    //      and, when the table allows it, 128 x 128 (tcgen05 kernel). ----
    const int G = std::max(1, t->sm_count);
    static const int env_penalty = [] { const char* e = getenv("AF_UNIT_PENALTY"); return e ? atoi(e) : 4; }();
    // cta0_extra: CTA 0 also materialises the residual stream and, with deferred RMSNorm scales, reads the
    // whole input vector alone -- its spans are shorter by that many tile-times
    auto build = [&](int tile_rows, int tile_cols, int penalty, int cta0_extra, std::vector<UnitDev>& units, int& grid,
                     long long* tiles_out) {
        std::vector<std::vector<UnitDev>> per_cta(G);
        int used = 0, first = 0;
        for (int ph = 0; ph < n_phases; ++ph) {
            const int strips = (g->x_len[ph] + tile_cols - 1) / tile_cols;
            long long total = 0;
            for (int i = 0; i < phase_len[ph]; ++i)
                total += (long long)strips * ((t->segs[seg_ids[first + i]].d_out + tile_rows - 1) / tile_rows);
            if (tiles_out) *tiles_out += total;
            const int Gp = (int)std::min<long long>(total, G);   // CTA 0 always owns tiles of every phase (it writes h_out)
            used = std::max(used, Gp);
            // Cost model of a span: its tiles + `penalty` tile-times for every strip boundary inside it
            // (a unit change restages the gated DOWN slab and refills the per-unit registers: ~4 us
            // against ~0.85 us per tile, profiles/r01c_chase_timeline.txt).  All CTAs meet at the phase
            // barrier, so spans are cut to equal COST, not equal tile count: the smallest per-CTA
            // budget that needs at most Gp spans, found by bisection.
            struct Strip { int sidx, slot, sp, rt, d_out; };
            std::vector<Strip> strips_v;
            for (int i = 0; i < phase_len[ph]; ++i) {
                const int sidx = seg_ids[first + i];
                const int d_out = t->segs[sidx].d_out;
                for (int sp = 0; sp < strips; ++sp) strips_v.push_back({sidx, first + i, sp, (d_out + tile_rows - 1) / tile_rows, d_out});
            }
            // Spans end at multiples of a fractional per-CTA budget (total cost / Gp), so every CTA gets
            // its share to within one tile; the total cost depends on how many spans cross a strip
            // boundary, which depends on the cut -- three fixed-point rounds settle it.
            // Share of the phase each CTA gets: equal, or the caller's measured shares (af_chain_create_weighted: an SM's
            // rate depends on where it sits -- its L2 die, its distance to the memory partitions -- by a few per cent,
            // the same in every launch; all CTAs meet at the phase barrier, so the slowest one sets the phase's time).
            std::vector<double> cum(Gp + 1, 0.0);
            for (int c = 0; c < Gp; ++c) cum[c + 1] = cum[c] + ((cta_share && c < n_cta) ? (double)cta_share[(size_t)ph * n_cta + c] : 1.0);
            for (int c = 1; c <= Gp; ++c) cum[c] *= (double)Gp / cum[Gp];     // in units of the equal share
            auto cut = [&](double budget, std::vector<std::vector<UnitDev>>* out) -> int {
                int cta = 0, crossings = 0;
                // cumulative cost of everything emitted so far; CTA 0 starts with its extra duties on the books,
                // but always keeps at least one tile (it is the one that writes h_out / the deferred scale)
                double cost = Gp > 1 ? std::min<double>(cta0_extra, std::max(0.0, std::floor(budget) - 1.0)) : 0.0;
                long long in_span = 0;                             // tiles the current span already holds
                for (const Strip& st : strips_v) {
                    int r = 0;
                    bool entered = false;
                    while (r < st.rt) {
                        const double span_end = cum[cta + 1] * budget;
                        if (!entered) {
                            entered = true;
                            if (in_span > 0) {   // the span continues into this strip: a unit change
                                cost += penalty;
                                ++crossings;
                            }
                        }
                        long long room = (long long)std::floor(span_end - cost + 1e-6);
                        if (room < 1 && cta == 0 && in_span == 0) room = 1;   // CTA 0 owns a tile of every phase (it writes h_out / the deferred scale)
                        if (room < 1) {
                            if (cta < Gp - 1) {
                                ++cta;
                                in_span = 0;
                                continue;
                            }
                            room = st.rt - r;   // the last CTA takes what is left
                        }
                        const int take = (int)std::min<long long>(st.rt - r, room);
                        if (out) {
                            const int row0 = r * tile_rows;
                            (*out)[cta].push_back({st.sidx, row0, std::min(take * tile_rows, st.d_out - row0), st.sp * tile_cols, ph, st.slot});
                        }
                        cost += take;
                        in_span += take;
                        r += take;
                    }
                }
                return crossings;
            };
            int crossings = 0;
            const long long extra = Gp > 1 ? cta0_extra : 0;
            for (int round = 0; round < 3; ++round) crossings = cut((double)(total + extra + (long long)penalty * crossings) / Gp, nullptr);
            cut((double)(total + extra + (long long)penalty * crossings) / Gp, &per_cta);
            first += phase_len[ph];
        }
        grid = used;
        size_t depth = 0;
        for (auto& v : per_cta) depth = std::max(depth, v.size());
        units.assign(depth * grid, UnitDev{0, 0, 0, 0, 0, 0});
        for (int c = 0; c < grid; ++c)
            for (size_t j = 0; j < per_cta[c].size(); ++j) units[j * grid + c] = per_cta[c][j];
    };
    std::vector<UnitDev> units, units_umma;
    build(kMR, kTN, env_penalty, 2, units, g->grid, &g->tiles);
    g->n_units = (int)units.size();
    bool umma = t->umma_ok;
    if (umma) {
        static const int env_penalty_u = [] { const char* e = getenv("AF_UNIT_PENALTY_UMMA"); return e ? atoi(e) : 2; }();
        // a 128 x 128 tile is 4x the bytes of the mma.sync kernel's: a unit change weighs about two tiles (swept 0 .. 3 on
        // Llama-2-7B: 5.59 / 5.53 / 5.50 / 5.53 ms per token)
        build(kUM, kUN, env_penalty_u, 2, units_umma, g->grid_umma, nullptr);
        g->n_units_umma = (int)units_umma.size();
    }
    cudaError_t e = cudaMalloc(&g->d_units, sizeof(UnitDev) * units.size());
    if (e == cudaSuccess) e = cudaMemcpy(g->d_units, units.data(), sizeof(UnitDev) * units.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && umma) e = cudaMalloc(&g->d_units_umma, sizeof(UnitDev) * units_umma.size());
    if (e == cudaSuccess && umma)
        e = cudaMemcpy(g->d_units_umma, units_umma.data(), sizeof(UnitDev) * units_umma.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_seg_yoff, sizeof(int) * yoff.size());
    if (e == cudaSuccess) e = cudaMemcpy(g->d_seg_yoff, yoff.data(), sizeof(int) * yoff.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        af_group_destroy(g);
        return fail(AF_ECUDA, std::string("group upload: ") + cudaGetErrorString(e));
    }
    *out = g;
    return AF_OK;
}

int af_group_create(af_table* t, const int32_t* seg_ids, int32_t n, af_group** out) {
    return af_chain_create(t, seg_ids, &n, 1, out);
}

int af_group_info(const af_group* g, int32_t* n_phases, int32_t* x_len, int32_t* y_rows, int32_t* n_units, int32_t* grid,
                  int64_t* tiles) {
    if (!g) return fail(AF_EVALUE, "group is NULL");
    if (n_phases) *n_phases = g->n_phases;
    for (int ph = 0; ph < g->n_phases; ++ph) {
        if (x_len) x_len[ph] = g->x_len[ph];
        if (y_rows) y_rows[ph] = g->y_rows[ph];
    }
    if (n_units) *n_units = g->n_units;
    if (grid) *grid = g->d_units_umma ? g->grid_umma : g->grid;   // the launch size: tcgen05 schedule when the table has one
    if (tiles) *tiles = g->tiles;
    return AF_OK;
}

int af_plan_build(af_table* t, const af_decision* prev_dev, const af_decision* cur_dev, int32_t max_k, float scale,
                  int32_t mode, void* stream) {
    if (!t) return fail(AF_EVALUE, "table is NULL");
    if (mode != AF_SWITCH_INPLACE && mode != AF_SWITCH_FROM_PRISTINE) return fail(AF_EVALUE, "unknown switch mode");
    if (max_k < 1 || max_k > AF_MAX_K) return fail(AF_EVALUE, "max_k outside [1, AF_MAX_K]");
    SwitchParams p{};
    p.from_pristine = mode == AF_SWITCH_FROM_PRISTINE;
    p.prev_dev = prev_dev;
    p.cur_dev = cur_dev;
    p.use_dev = 1;
    p.scale = scale;
    p.n_experts_limit = t->min_experts;
    p.err_flag = t->err_word;
    const int bound = (p.from_pristine || !prev_dev ? 0 : max_k) + (cur_dev ? max_k : 0);
    p.max_blocks = std::min(bound, kMaxBlocks);
    plan_build_kernel<<<1, 32, 0, as_stream(stream)>>>(p, t->d_plan);
    AF_LAUNCH_CHECK("plan_build_kernel");
    return AF_OK;
}

int af_switch_gemv_chain(af_group* g, const af_decision* prev_dev, const af_decision* cur_dev, int32_t max_k, float scale,
                         int32_t mode, const af_gemv_phase* phases, int32_t n_phases, int32_t* phase_done_dev, int32_t flags,
                         void* stream) {
    const int pdl = flags & AF_CHAIN_PDL;
    if (!g) return fail(AF_EVALUE, "group is NULL");
    af_table* t = g->table;
    if (mode != AF_SWITCH_INPLACE && mode != AF_SWITCH_FROM_PRISTINE) return fail(AF_EVALUE, "unknown switch mode");
    if (mode == AF_SWITCH_FROM_PRISTINE && !t->has_pristine)
        return fail(AF_ESTATE, "FROM_PRISTINE needs a pristine copy of every segment");
    if (!phases || n_phases != g->n_phases) return fail(AF_EDIM, "one af_gemv_phase per phase of the chain");
    if (n_phases > 1 && !phase_done_dev) return fail(AF_EVALUE, "a chain of several phases needs its phase_done counters");
    if (g->n_peers > 0 && ((g->reduce_mask >> (n_phases - 1)) & 1) && !phase_done_dev)
        return fail(AF_EVALUE, "a last phase that is pushed to the peers reports on phase_done[n_phases - 1]: counters needed");
    for (int ph = 0; ph < n_phases; ++ph) {
        const af_gemv_phase& f = phases[ph];
        if (f.prologue < AF_PRO_NONE || f.prologue > AF_PRO_RMSNORM_DEFERRED) return fail(AF_EVALUE, "unknown prologue");
        if ((f.prologue == AF_PRO_RMSNORM || f.prologue == AF_PRO_RMSNORM_DEFERRED) && !f.norm_w)
            return fail(AF_EVALUE, "RMSNorm prologue needs its weight vector");
        if (f.prologue == AF_PRO_RMSNORM_DEFERRED && !f.inv_out) return fail(AF_EVALUE, "deferred RMSNorm needs inv_out");
        if ((f.xin == nullptr) == (f.acc_in == nullptr)) return fail(AF_EVALUE, "exactly one of xin / acc_in must be given");
        if (!f.acc_out) return fail(AF_EVALUE, "acc_out is NULL");
        if (reinterpret_cast<uintptr_t>(f.acc_out) % 8 != 0 || reinterpret_cast<uintptr_t>(f.acc_in) % 16 != 0)
            return fail(AF_EDIM, "fixed-point accumulators must be 8-byte aligned (16-byte as an input)");
        if (reinterpret_cast<uintptr_t>(f.xin) % 8 != 0 || reinterpret_cast<uintptr_t>(f.res) % 8 != 0 ||
            reinterpret_cast<uintptr_t>(f.h_out) % 8 != 0 || g->x_len[ph] % 2 != 0)
            return fail(AF_EDIM, "input vectors must be 8-byte aligned and of even length");
        if (f.h_out && (f.h_out == f.xin || f.h_out == f.res)) return fail(AF_EALIAS, "h_out aliases an input vector");
    }
    const bool use_dev = prev_dev || cur_dev;
    if (use_dev && (max_k < 1 || max_k > AF_MAX_K)) return fail(AF_EVALUE, "max_k outside [1, AF_MAX_K]");
    const bool from_pristine = mode == AF_SWITCH_FROM_PRISTINE;

    MmaParams mp{};
    SwitchParams& p = mp.base;
    p.segs = t->d_segs;
    p.units = g->d_units;
    p.n_units = g->n_units;
    p.from_pristine = from_pristine;
    p.prev_dev = prev_dev;
    p.cur_dev = cur_dev;
    p.use_dev = use_dev ? 1 : 0;
    p.scale = scale;
    p.n_experts_limit = t->min_experts;
    p.err_flag = t->err_word;
    p.host_plan.n_blocks = 0;  // no decision at all: a plain GEMV over the live weights
    p.plan_dev = (use_dev && (flags & AF_CHAIN_PLAN_PREBUILT)) ? t->d_plan : nullptr;
    const int n_blocks_bound = use_dev ? ((from_pristine || !prev_dev ? 0 : max_k) + (cur_dev ? max_k : 0)) : 0;
    p.max_blocks = std::min(n_blocks_bound, kMaxBlocks);
    const int s_bound = n_blocks_bound * t->max_rank;
    const bool umma_launch = g->d_units_umma && s_bound <= std::min(kUmmaMaxRanksChain, umma_rank_limit(t));
    if (s_bound > kMmaMaxKS * 16 && !umma_launch)
        return fail(AF_EVALUE, "the fused switch + GEMV holds at most 64 stacked ranks (256 on the tcgen05 path)");
    const int S = t->n_segments;
    mp.tmaps_ld = t->d_maps + (size_t)(from_pristine ? 3 : 2) * S;
    mp.tmaps_st = t->d_maps + (size_t)2 * S;
    mp.tmaps_up = t->d_maps + (size_t)4 * S;
    for (int ph = 0; ph < n_phases; ++ph) {
        const af_gemv_phase& f = phases[ph];
        GemvParams& gv = mp.gv[ph];
        gv.xin = f.xin;
        gv.acc_in = reinterpret_cast<const long long*>(f.acc_in);
        gv.res = f.res;
        gv.h_out = f.h_out;
        gv.norm_w = f.norm_w;
        gv.eps = f.eps;
        gv.prologue = f.prologue;
        gv.x_len = g->x_len[ph];
        gv.acc_out = reinterpret_cast<unsigned long long*>(f.acc_out);
        gv.inv_out = f.inv_out;
        gv.inv_in = f.inv_in;
    }
    mp.n_phases = n_phases;
    mp.phase_done = phase_done_dev;
    mp.seg_yoff = g->d_seg_yoff;
    mp.mixed_rank = t->mixed_rank ? 1 : 0;
    mp.n_chain_segs = (int)g->segs.size();
    for (size_t i = 0; i < g->segs.size(); ++i) mp.chain_segs[i] = g->segs[i];
    mp.pdl = (pdl && g_pdl.load()) ? 1 : 0;
    static const int env_dbg = [] { const char* e = getenv("AF_DBG"); return e ? atoi(e) : 0; }();
    mp.dbg = env_dbg ^ 24;
    const int ks_tl = std::max(1, (s_bound + 15) / 16);
    if (g_timeline && g_timeline_left > 0 && (ks_tl == 2 || umma_launch)) {  // mma.sync: the probe is compiled into the KS = 2 hi/lo variant only
        mp.timeline = g_timeline;
        g_timeline += g_timeline_stride;
        --g_timeline_left;
    }
    const int ks = std::max(1, (s_bound + 15) / 16);
    const bool ba = t->rank16 && ks > 2 && !g_force_hilo;
    cudaStream_t st = as_stream(stream);
    if (env_dbg & 4) {  // experiment: the plain switch kernel on this group's schedule (no GEMV at all)
        if (ks == 2) return launch_mma<2, false, false>(mp, g->grid, st);
    }
    // tcgen05 path (env AF_UMMA=1 while it is being validated): rank-8 tables of 128-multiples
    for (int ph = 0; ph < n_phases; ++ph)
        if ((phases[ph].prologue == AF_PRO_RMSNORM_DEFERRED || phases[ph].inv_in) && !umma_launch)
            return fail(AF_ESTATE, "deferred RMSNorm scales are implemented by the tcgen05 kernel only (table info: umma_path)");
    if (g->n_peers > 0 && !umma_launch)
        return fail(AF_ESTATE, "peer accumulation (af_group_set_peers) is implemented by the tcgen05 kernel only (table info: umma_path)");
    if (umma_launch) {
        p.units = g->d_units_umma;
        p.n_units = g->n_units_umma;
        mp.tmaps_ld = t->d_maps + (size_t)(from_pristine ? 6 : 5) * S;
        mp.tmaps_st = t->d_maps + (size_t)5 * S;
        mp.tmaps_up = t->d_maps + (size_t)7 * S;
        mp.n_peers = g->n_peers;
        mp.reduce_mask = g->reduce_mask;
        for (int w = 0; w < g->n_peers; ++w) mp.peer_off[w] = g->peer_off[w];
        return dispatch_umma<true>(t, s_bound, mp, g->grid_umma, st);
    }
    if (mp.timeline && ks == 2) return launch_mma<2, false, true, true>(mp, g->grid, st);
    switch (ks) {
        case 1: return launch_mma<1, false, true>(mp, g->grid, st);
        case 2: return launch_mma<2, false, true>(mp, g->grid, st);
        case 3: return ba ? launch_mma<3, true, true>(mp, g->grid, st) : launch_mma<3, false, true>(mp, g->grid, st);
        default: return ba ? launch_mma<4, true, true>(mp, g->grid, st) : launch_mma<4, false, true>(mp, g->grid, st);
    }
}

int af_group_set_peers(af_group* g, int32_t n_peers, const int64_t* peer_offset_bytes, int32_t reduce_phase_mask) {
    if (!g) return fail(AF_EVALUE, "group is NULL");
    if (n_peers == 0) {   // back to a single rank
        g->n_peers = 0;
        g->reduce_mask = 0;
        return AF_OK;
    }
    if (n_peers < 1 || n_peers > 8) return fail(AF_EVALUE, "1 .. 8 peers (this rank included)");
    if (!peer_offset_bytes) return fail(AF_EVALUE, "peer offsets are NULL");
    if (!g->d_units_umma) return fail(AF_ESTATE, "peer accumulation needs the tcgen05 path (table info: umma_path)");
    if (reduce_phase_mask < 0 || reduce_phase_mask >= (1 << g->n_phases)) return fail(AF_EVALUE, "reduce mask names a phase the chain does not have");
    int zeros = 0;
    for (int w = 0; w < n_peers; ++w) {
        if (peer_offset_bytes[w] % 8 != 0) return fail(AF_EDIM, "peer offsets must keep the 8-byte alignment of the accumulators");
        zeros += peer_offset_bytes[w] == 0;
        for (int v = 0; v < w; ++v)
            if (peer_offset_bytes[v] == peer_offset_bytes[w]) return fail(AF_EALIAS, "two peers at the same address");
    }
    if (zeros != 1) return fail(AF_EVALUE, "the list must contain this rank itself (offset 0) exactly once");
    g->n_peers = n_peers;
    g->reduce_mask = reduce_phase_mask;
    for (int w = 0; w < n_peers; ++w) g->peer_off[w] = peer_offset_bytes[w];
    return AF_OK;
}

static int peer_list(int32_t n_peers, const int64_t* peer_offset_bytes, PeerList& pl) {
    if (n_peers < 1 || n_peers > 8 || !peer_offset_bytes) return fail(AF_EVALUE, "1 .. 8 peers (this rank included)");
    pl.n = n_peers;
    for (int w = 0; w < n_peers; ++w) {
        if (peer_offset_bytes[w] % 4 != 0) return fail(AF_EDIM, "peer offsets must keep the counters aligned");
        pl.off[w] = peer_offset_bytes[w];
    }
    return AF_OK;
}

int af_peer_barrier(int32_t* counter_dev, int32_t* epoch_dev, int32_t n_peers, const int64_t* peer_offset_bytes,
                    int32_t* err_flag_dev, void* stream) {
    if (!counter_dev || !epoch_dev) return fail(AF_EVALUE, "counter / epoch is NULL");
    PeerList pl{};
    if (int rc = peer_list(n_peers, peer_offset_bytes, pl)) return rc;
    peer_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(counter_dev, epoch_dev, pl, err_flag_dev);
    AF_LAUNCH_CHECK("peer_barrier_kernel");
    return AF_OK;
}

int af_peer_bcast(const void* src_dev, void* slot_dev, void* dst_dev, int32_t bytes, int32_t is_root, int32_t* counter_dev,
                  int32_t* epoch_dev, int32_t n_peers, const int64_t* peer_offset_bytes, int32_t* err_flag_dev, void* stream) {
    if (!slot_dev || !dst_dev || !counter_dev || !epoch_dev || (is_root && !src_dev)) return fail(AF_EVALUE, "NULL argument");
    if (bytes < 4 || bytes > 4096 || bytes % 4 != 0) return fail(AF_EDIM, "a broadcast record is 4 .. 4096 bytes, a multiple of 4");
    PeerList pl{};
    if (int rc = peer_list(n_peers, peer_offset_bytes, pl)) return rc;
    peer_bcast_kernel<<<1, 128, 0, as_stream(stream)>>>(static_cast<const uint32_t*>(src_dev), static_cast<uint32_t*>(slot_dev),
                                                         static_cast<uint32_t*>(dst_dev), bytes / 4, is_root ? 1 : 0, counter_dev, epoch_dev, pl,
                                                         err_flag_dev);
    AF_LAUNCH_CHECK("peer_bcast_kernel");
    return AF_OK;
}

int af_peer_argmax(const float* val_dev, const int32_t* idx_dev, void* slots_dev, int32_t my_slot, int32_t* counter_dev, int32_t* epoch_dev,
                   int32_t n_peers, const int64_t* peer_offset_bytes, int32_t* out_idx_dev, int32_t* err_flag_dev, void* stream) {
    if (!val_dev || !idx_dev || !slots_dev || !counter_dev || !epoch_dev || !out_idx_dev) return fail(AF_EVALUE, "NULL argument");
    if (reinterpret_cast<uintptr_t>(slots_dev) % 8 != 0) return fail(AF_EDIM, "the pair slots are 8-byte words");
    PeerList pl{};
    if (int rc = peer_list(n_peers, peer_offset_bytes, pl)) return rc;
    if (my_slot < 0 || my_slot >= n_peers) return fail(AF_EVALUE, "my_slot outside [0, n_peers)");
    for (int w = 0; w < n_peers; ++w)
        if (pl.off[w] % 8 != 0) return fail(AF_EDIM, "peer offsets must keep the 8-byte alignment of the pair slots");
    peer_argmax_kernel<<<1, 32, 0, as_stream(stream)>>>(val_dev, idx_dev, static_cast<unsigned long long*>(slots_dev), my_slot, counter_dev,
                                                        epoch_dev, pl, out_idx_dev, err_flag_dev);
    AF_LAUNCH_CHECK("peer_argmax_kernel");
    return AF_OK;
}

int af_peer_wait(const int32_t* counter_dev, int32_t target, int32_t* err_flag_dev, void* stream) {
    if (!counter_dev) return fail(AF_EVALUE, "counter is NULL");
    peer_wait_kernel<<<1, 32, 0, as_stream(stream)>>>(counter_dev, target, err_flag_dev);
    AF_LAUNCH_CHECK("peer_wait_kernel");
    return AF_OK;
}

int af_switch_gemv(af_group* g, const af_decision* prev_dev, const af_decision* cur_dev, int32_t max_k, float scale,
                   int32_t mode, const float* xin, const int64_t* acc_in, const float* res, float* h_out, int32_t prologue,
                   const float* norm_w, float eps, int64_t* acc_out, int32_t pdl, void* stream) {
    af_gemv_phase f{};
    f.xin = xin;
    f.acc_in = acc_in;
    f.res = res;
    f.h_out = h_out;
    f.norm_w = norm_w;
    f.acc_out = acc_out;
    f.eps = eps;
    f.prologue = prologue;
    f.inv_out = nullptr;
    f.inv_in = nullptr;
    return af_switch_gemv_chain(g, prev_dev, cur_dev, max_k, scale, mode, &f, 1, nullptr, pdl, stream);
}

int af_set_timeline(uint64_t* buffer_dev, int32_t n_launches, int64_t stride_elems) {
    g_timeline = reinterpret_cast<unsigned long long*>(buffer_dev);
    g_timeline_left = buffer_dev ? n_launches : 0;
    g_timeline_stride = stride_elems;
    return AF_OK;
}

int af_accum_to_f32(const int64_t* acc, const float* res, float* out, int32_t n, void* stream) {
    if (n < 0 || !acc || !out) return fail(AF_EVALUE, "NULL argument");
    if (n == 0) return AF_OK;
    accum_to_f32_kernel<<<std::max(1, std::min((n + 255) / 256, 64)), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const long long*>(acc), res, out, n);
    AF_LAUNCH_CHECK("accum_to_f32_kernel");
    return AF_OK;
}

// ------------------------------------------------------------------ router ----

int af_pregate(const void* router_w, int32_t w_dtype, int32_t n_experts, int32_t d, const void* x, int32_t x_dtype,
               const int32_t* token_dev, int32_t k, af_decision* out_dev, float* logits_dev, void* stream) {
    // routing.py:57-58: k first
    if (n_experts < 1 || n_experts > kRouterMaxExperts) return fail(AF_EDIM, "router supports 1..256 experts");
    if (k < 1 || k > n_experts) return fail(AF_EVALUE, "k=" + std::to_string(k) + " must be in [1, " + std::to_string(n_experts) + "]");
    if (k > AF_MAX_K) return fail(AF_EVALUE, "k exceeds AF_MAX_K");
    if (d < 1) return fail(AF_EDIM, "hidden size must be positive");
    if (!router_w || !x || !out_dev) return fail(AF_EVALUE, "NULL argument");
    cudaStream_t st = as_stream(stream);
#define AF_PREGATE(WT, XT)                                                                                           \
    pregate_kernel<WT, XT><<<1, kRouterThreads, 0, st>>>(reinterpret_cast<const WT*>(router_w), n_experts, d,          \
                                                         reinterpret_cast<const XT*>(x), token_dev, k, out_dev, logits_dev)
    if (w_dtype == AF_BF16 && x_dtype == AF_BF16) AF_PREGATE(__nv_bfloat16, __nv_bfloat16);
    else if (w_dtype == AF_BF16 && x_dtype == AF_F32) AF_PREGATE(__nv_bfloat16, float);
    else if (w_dtype == AF_F32 && x_dtype == AF_BF16) AF_PREGATE(float, __nv_bfloat16);
    else if (w_dtype == AF_F32 && x_dtype == AF_F32) AF_PREGATE(float, float);
    else return fail(AF_EPRECISION, "unknown precision tag");
#undef AF_PREGATE
    AF_LAUNCH_CHECK("pregate_kernel");
    return AF_OK;
}

// ------------------------------------------------------------------ decode ----

int af_gemv(const void* w, int32_t w_dtype, int32_t rows, int32_t cols, int64_t ld, const float* x, float* out,
            int32_t epilogue, const float* res, void* stream) {
    if (rows < 0 || cols < 0 || ld < cols) return fail(AF_EDIM, "bad GEMV shape");
    if (epilogue < AF_EPI_NONE || epilogue > AF_EPI_RESIDUAL) return fail(AF_EVALUE, "unknown epilogue");
    if (epilogue != AF_EPI_NONE && !res) return fail(AF_EVALUE, "epilogue needs a residual vector");
    if (w_dtype != AF_BF16 && w_dtype != AF_F32) return fail(AF_EPRECISION, "unknown precision tag");
    if (rows == 0) return AF_OK;
    if (out == x) return fail(AF_EALIAS, "GEMV output aliases its input");
    const DeviceInfo& di = device_info();
    const int smem = cols * 4;
    if (smem > di.max_smem_optin) return fail(AF_EDIM, "GEMV input vector does not fit in shared memory");
    cudaStream_t st = as_stream(stream);
    const int rows_per_cta = (kGemvThreads / 32) * kRowsPerWarp;
    const int grid = std::max(1, std::min((rows + rows_per_cta - 1) / rows_per_cta, di.sm_count * 8));
    if (w_dtype == AF_BF16) {
        if (smem > 48 * 1024) AF_CUDA_TRY(cudaFuncSetAttribute(gemv_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        gemv_kernel<__nv_bfloat16><<<grid, kGemvThreads, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(w), rows, cols, ld, x, out, epilogue, res);
    } else {
        if (smem > 48 * 1024) AF_CUDA_TRY(cudaFuncSetAttribute(gemv_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        gemv_kernel<float><<<grid, kGemvThreads, smem, st>>>(reinterpret_cast<const float*>(w), rows, cols, ld, x, out, epilogue, res);
    }
    AF_LAUNCH_CHECK("gemv_kernel");
    return AF_OK;
}

int af_gemv_t(const void* w, int32_t w_dtype, int32_t rows, int32_t cols, int64_t ld, const float* x, float* out,
              void* stream) {
    if (rows < 0 || cols < 0 || ld < cols) return fail(AF_EDIM, "bad GEMV shape");
    if (w_dtype != AF_BF16 && w_dtype != AF_F32) return fail(AF_EPRECISION, "unknown precision tag");
    if (cols == 0) return AF_OK;
    cudaStream_t st = as_stream(stream);
    const int grid = (cols + kGemvTCols - 1) / kGemvTCols;
    if (w_dtype == AF_BF16)
        gemv_t_kernel<__nv_bfloat16><<<grid, kGemvTThreads, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(w), rows, cols, ld, x, out);
    else
        gemv_t_kernel<float><<<grid, kGemvTThreads, 0, st>>>(reinterpret_cast<const float*>(w), rows, cols, ld, x, out);
    AF_LAUNCH_CHECK("gemv_t_kernel");
    return AF_OK;
}

int af_argmax(const float* v, int32_t n, int32_t* out_dev, void* stream) {
    if (n < 1 || !v || !out_dev) return fail(AF_EDIM, "argmax of an empty vector");
    argmax_kernel<<<1, 1024, 0, as_stream(stream)>>>(v, n, out_dev);
    AF_LAUNCH_CHECK("argmax_kernel");
    return AF_OK;
}

int af_embed(const void* table, int32_t dtype, int32_t d, const int32_t* token_dev, float* out, void* stream) {
    if (d < 1 || !table || !token_dev || !out) return fail(AF_EDIM, "bad embed arguments");
    const int grid = std::max(1, std::min((d + 255) / 256, 64));
    if (dtype == AF_BF16)
        embed_kernel<__nv_bfloat16><<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<const __nv_bfloat16*>(table), d, token_dev, out);
    else if (dtype == AF_F32)
        embed_kernel<float><<<grid, 256, 0, as_stream(stream)>>>(reinterpret_cast<const float*>(table), d, token_dev, out);
    else
        return fail(AF_EPRECISION, "unknown precision tag");
    AF_LAUNCH_CHECK("embed_kernel");
    return AF_OK;
}

// ------------------------------------------------------------------ Llama block ----

int af_gemv_fused(const void* w, int32_t rows, int32_t cols, int64_t ld, const float* x, float* out, int32_t prologue,
                  const float* norm_w, float eps, int32_t epilogue, const float* res, void* stream) {
    if (rows < 0 || cols < 1 || ld < cols) return fail(AF_EDIM, "bad GEMV shape");
    if (cols % 8 != 0 || ld % 8 != 0 || (reinterpret_cast<uintptr_t>(w) & 15) != 0)
        return fail(AF_EDIM, "fused GEMV needs 16-byte aligned bf16 rows (cols % 8 == 0)");
    if (prologue < AF_PRO_NONE || prologue > AF_PRO_SILU_MUL) return fail(AF_EVALUE, "unknown prologue");
    if (prologue == AF_PRO_RMSNORM && !norm_w) return fail(AF_EVALUE, "RMSNorm prologue needs its weight vector");
    if (epilogue < AF_EPI_NONE || epilogue > AF_EPI_RESIDUAL) return fail(AF_EVALUE, "unknown epilogue");
    if (epilogue != AF_EPI_NONE && !res) return fail(AF_EVALUE, "epilogue needs a residual vector");
    if (!w || !x || !out) return fail(AF_EVALUE, "NULL argument");
    if (out == x) return fail(AF_EALIAS, "GEMV output aliases its input");
    if (rows == 0) return AF_OK;
    const DeviceInfo& di = device_info();
    const int xs_bytes = cols * 4;
    if ((reinterpret_cast<uintptr_t>(x) & 15) != 0 || (norm_w && (reinterpret_cast<uintptr_t>(norm_w) & 15) != 0) || cols % 4 != 0)
        return fail(AF_EDIM, "fused GEMV needs 16-byte aligned f32 vectors");
    cudaLaunchConfig_t cfg{};
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl.load() ? 1 : 0;
    const __nv_bfloat16* wp = reinterpret_cast<const __nv_bfloat16*>(w);
    const int variant = g_gemv_variant.load();
    if (variant == 0) {
        // register-streamed kernel: even split of the rows over SMs x resident CTAs
        if (xs_bytes + 1024 > di.max_smem_optin) return fail(AF_EDIM, "GEMV input vector does not fit in shared memory");
        static PerDevice configured;
        if (xs_bytes > std::max(48 * 1024, configured.cur())) {
            AF_CUDA_TRY(cudaFuncSetAttribute(gemv_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, xs_bytes));
            configured.cur() = xs_bytes;
        }
        static PerDevice occ_smem_d, occ_d;
        int& occ_smem = occ_smem_d.cur();
        int& occ = occ_d.cur();
        if (occ_smem != xs_bytes + 1) {
            AF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_fused_kernel, kGemvFThreads, xs_bytes));
            occ_smem = xs_bytes + 1;
        }
        cfg.gridDim = dim3(std::max(1, std::min(rows, di.sm_count * std::max(1, std::min(occ, 8)))));
        cfg.blockDim = dim3(kGemvFThreads);
        cfg.dynamicSmemBytes = xs_bytes;
        AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemv_fused_kernel, wp, (int)rows, (int)cols, (long long)ld, x, out, (int)prologue,
                                       norm_w, eps, (int)epilogue, res));
    } else {
        // TMA-ring kernel: variant 1 = 2 KB copies / 1 producer, 2 = 2 KB / 2 producers, 3 = 4 KB / 1, 4 = 4 KB / 2
        const int ch = (variant >= 3) ? 2048 : 1024;
        const int stage = kGvWarps * ch * 2;
        // The footprint is held to half an SM when that still leaves >= 3 stages, so that under
        // programmatic dependent launch the next GEMV's CTA is co-resident and fills its ring
        // while this kernel drains.
        const int half_sm = (di.max_smem_optin - 2048) / 2;
        int n_stages = (half_sm - xs_bytes) / stage;
        if (n_stages < 3 || g_gemv_full_sm.load()) n_stages = (di.max_smem_optin - 2048 - xs_bytes) / stage;
        n_stages = std::min(n_stages, kGvMaxStages);
        if (n_stages < 2) return fail(AF_EDIM, "GEMV input vector does not fit in shared memory");
        const int smem = n_stages * stage + xs_bytes;
        cfg.gridDim = dim3(std::max(1, std::min((rows + kGvWarps - 1) / kGvWarps, di.sm_count)));
        cfg.dynamicSmemBytes = smem;
#define AF_GV_LAUNCH(CH, NP)                                                                                              \
    do {                                                                                                                  \
        static PerDevice configured;                                                                                      \
        if (smem > configured.cur()) {                                                                                    \
            AF_CUDA_TRY(cudaFuncSetAttribute(gemv_tma_kernel<CH, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
            configured.cur() = smem;                                                                                      \
        }                                                                                                                 \
        cfg.blockDim = dim3(kGvWarps * 32 + 32 * NP);                                                                     \
        AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemv_tma_kernel<CH, NP>, wp, (int)rows, (int)cols, (long long)ld, x, out,     \
                                       (int)prologue, norm_w, eps, (int)epilogue, res, n_stages));                        \
    } while (0)
        if (variant == 1) AF_GV_LAUNCH(1024, 1);
        else if (variant == 2) AF_GV_LAUNCH(1024, 2);
        else if (variant == 3) AF_GV_LAUNCH(2048, 1);
        else AF_GV_LAUNCH(2048, 2);
#undef AF_GV_LAUNCH
    }
    AF_LAUNCH_CHECK("gemv_tma_kernel");
    return AF_OK;
}

static int attn_decode_impl(const float* qkv, const long long* qkv_fix, const float* qkv_scale, void* k_cache, void* v_cache,
                            const float* cos_table, const float* sin_table, const int32_t* pos_dev, int32_t n_heads,
                            int32_t n_kv_heads, int32_t head_dim, int32_t max_seq, int32_t n_split, float* workspace,
                            int32_t* tickets, float* out, void* stream);

int af_gemv_chain(const af_gv_phase* phases, int32_t n_phases, int32_t* phase_done_dev, int32_t* err_flag_dev, int32_t pdl,
                  void* stream) {
    if (!phases || n_phases < 1 || n_phases > kGcMaxPhases) return fail(AF_EVALUE, "a GEMV chain has 1..4 phases");
    if (n_phases > 1 && !phase_done_dev) return fail(AF_EVALUE, "a chain of several phases needs its phase_done counters");
    const DeviceInfo& di = device_info();
    if (!di.ok) return fail(AF_ECUDA, "no CUDA device");
    GcParams gp{};
    int max_cols = 0;
    long long max_rows = 0;
    for (int i = 0; i < n_phases; ++i) {
        const af_gv_phase& f = phases[i];
        if (f.rows < 1 || f.cols < 1 || f.ld < f.cols) return fail(AF_EDIM, "bad GEMV shape");
        if (f.cols % 8 != 0 || f.ld % 8 != 0 || (reinterpret_cast<uintptr_t>(f.w) & 15) != 0)
            return fail(AF_EDIM, "chained GEMV needs 16-byte aligned bf16 rows (cols % 8 == 0)");
        if (f.prologue < AF_PRO_NONE || f.prologue > AF_PRO_SILU_MUL) return fail(AF_EVALUE, "unknown prologue");
        if (f.prologue == AF_PRO_RMSNORM && !f.norm_w) return fail(AF_EVALUE, "RMSNorm prologue needs its weight vector");
        if (f.epilogue < AF_EPI_NONE || f.epilogue > AF_EPI_RESIDUAL) return fail(AF_EVALUE, "unknown epilogue");
        if (f.epilogue != AF_EPI_NONE && !f.res) return fail(AF_EVALUE, "epilogue needs a residual vector");
        if (!f.w || !f.x || !f.out) return fail(AF_EVALUE, "NULL argument");
        if (f.out == f.x) return fail(AF_EALIAS, "GEMV output aliases its input");
        if ((reinterpret_cast<uintptr_t>(f.x) & 15) != 0 || (f.norm_w && (reinterpret_cast<uintptr_t>(f.norm_w) & 15) != 0))
            return fail(AF_EDIM, "chained GEMV needs 16-byte aligned f32 vectors");
        GcPhase& g = gp.ph[i];
        g.w = reinterpret_cast<const __nv_bfloat16*>(f.w);
        g.rows = f.rows;
        g.cols = f.cols;
        g.ld = f.ld;
        g.x = f.x;
        g.out = f.out;
        g.res = f.res;
        g.norm_w = f.norm_w;
        g.eps = f.eps;
        g.prologue = f.prologue;
        g.epilogue = f.epilogue;
        max_cols = std::max(max_cols, (int)f.cols);
        max_rows = std::max<long long>(max_rows, f.rows);
    }
    const int xs_bytes = max_cols * 4;
    int n_stages = (di.max_smem_optin - 1024 - xs_bytes) / kGcStage;
    n_stages = std::min(n_stages, kGcMaxStages);
    if (n_stages < 2) return fail(AF_EDIM, "GEMV input vector does not fit in shared memory next to the weight ring");
    const int smem = n_stages * kGcStage + xs_bytes;
    static PerDevice configured;
    if (smem > configured.cur()) {
        AF_CUDA_TRY(cudaFuncSetAttribute(gemv_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        configured.cur() = smem;
    }
    if (n_phases > 1) {   // co-residency of the whole grid (in-kernel phase barriers), checked once per device
        static PerDevice occ_checked;
        if (occ_checked.cur() < smem) {
            int per_sm = 0;
            AF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemv_chain_kernel, kGcThreads, smem));
            if (per_sm < 1) return fail(AF_ESTATE, "a chained GEMV launch needs one resident CTA per SM; this device cannot hold it");
            occ_checked.cur() = smem;
        }
    }
    gp.n_phases = n_phases;
    gp.phase_done = phase_done_dev;
    gp.n_stages = n_stages;
    gp.pdl = (pdl && g_pdl.load()) ? 1 : 0;
    gp.err_flag = err_flag_dev;
    cudaLaunchConfig_t cfg{};
    // every CTA takes part in the phase barriers: the grid is one CTA per SM, all co-resident
    cfg.gridDim = dim3(di.sm_count);
    cfg.blockDim = dim3(kGcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = gp.pdl ? 1 : 0;
    AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemv_chain_kernel, gp));
    AF_LAUNCH_CHECK("gemv_chain_kernel");
    return AF_OK;
}

int af_forward_validate(const af_fw_phase* ph, int32_t n_phases, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                        int32_t* max_cols_out) {
    if (!ph || n_phases < 1) return fail(AF_EVALUE, "a forward needs at least one phase");
    if (n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads != 0) return fail(AF_EDIM, "heads must be a multiple of kv heads");
    if (head_dim != 64 && head_dim != 128) return fail(AF_EDIM, "the persistent forward takes head_dim 64 or 128");
    static_assert(sizeof(af_fw_phase) == sizeof(FwPhase), "af_fw_phase mirrors FwPhase");
    int max_cols = 0;
    for (int i = 0; i < n_phases; ++i) {
        const af_fw_phase& f = ph[i];
        if (f.kind == AF_FW_GEMV) {
            if (f.rows < 1 || f.cols < 1 || f.ld < f.cols) return fail(AF_EDIM, "bad GEMV shape");
            if (f.cols % 8 != 0 || f.ld % 8 != 0 || (reinterpret_cast<uintptr_t>(f.w) & 15) != 0)
                return fail(AF_EDIM, "GEMV phases need 16-byte aligned bf16 rows (cols % 8 == 0)");
            if (f.prologue < AF_PRO_NONE || f.prologue > AF_PRO_SILU_MUL) return fail(AF_EVALUE, "unknown prologue");
            if (f.prologue == AF_PRO_RMSNORM && !f.norm_w) return fail(AF_EVALUE, "RMSNorm prologue needs its weight vector");
            if (f.epilogue < AF_EPI_NONE || f.epilogue > AF_EPI_RESIDUAL) return fail(AF_EVALUE, "unknown epilogue");
            if (f.epilogue != AF_EPI_NONE && !f.res) return fail(AF_EVALUE, "epilogue needs a residual vector");
            if (!f.w || !f.x || !f.out) return fail(AF_EVALUE, "NULL argument");
            if (f.out == f.x) return fail(AF_EALIAS, "GEMV output aliases its input");
            if ((reinterpret_cast<uintptr_t>(f.x) & 15) != 0 || (f.norm_w && (reinterpret_cast<uintptr_t>(f.norm_w) & 15) != 0))
                return fail(AF_EDIM, "GEMV phases need 16-byte aligned f32 vectors");
            max_cols = std::max(max_cols, (int)f.cols);
        } else if (f.kind == AF_FW_ATTN_PARTIAL) {
            if (!f.x || !f.k_cache || !f.v_cache) return fail(AF_EVALUE, "attention phase: NULL argument");
            if ((reinterpret_cast<uintptr_t>(f.k_cache) & 15) != 0 || (reinterpret_cast<uintptr_t>(f.v_cache) & 15) != 0)
                return fail(AF_EDIM, "KV caches must be 16-byte aligned");
        } else if (f.kind == AF_FW_ATTN_COMBINE) {
            if (!f.out) return fail(AF_EVALUE, "attention combine: NULL output");
            if (i == 0 || ph[i - 1].kind != AF_FW_ATTN_PARTIAL) return fail(AF_EVALUE, "an attention combine follows its partials phase");
        } else {
            return fail(AF_EVALUE, "unknown phase kind");
        }
    }
    if (max_cols_out) *max_cols_out = max_cols;
    return AF_OK;
}

int af_forward_persistent(const af_fw_phase* phases_dev, int32_t n_phases, int32_t max_cols, const float* cos_table,
                          const float* sin_table, const int32_t* pos_dev, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                          int32_t max_seq, float* workspace, int32_t* phase_done_dev, int32_t* err_flag_dev, int32_t pdl, void* stream) {
    if (!phases_dev || n_phases < 1 || !phase_done_dev) return fail(AF_EVALUE, "NULL argument");
    if (head_dim != 64 && head_dim != 128) return fail(AF_EDIM, "the persistent forward takes head_dim 64 or 128");
    if (n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads != 0 || max_seq < 1) return fail(AF_EDIM, "bad attention geometry");
    if (!cos_table || !sin_table || !pos_dev || !workspace) return fail(AF_EVALUE, "NULL argument");
    if (max_cols < 8) return fail(AF_EDIM, "max_cols comes from af_forward_validate");
    const DeviceInfo& di = device_info();
    if (!di.ok) return fail(AF_ECUDA, "no CUDA device");
    // the input-vector area doubles as the attention teams' merge buffers
    const int xs_bytes = std::max(max_cols * 4, kFwTeams * kFwTeamWarps * (head_dim + 2) * 4);
    int n_stages = (di.max_smem_optin - 2048 - xs_bytes) / kGcStage;
    n_stages = std::min(n_stages, kGcMaxStages);
    if (n_stages < 2) return fail(AF_EDIM, "GEMV input vector does not fit in shared memory next to the weight ring");
    const int smem = n_stages * kGcStage + xs_bytes;
    static PerDevice configured;
    if (smem > configured.cur()) {
        AF_CUDA_TRY(cudaFuncSetAttribute(forward_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int per_sm = 0;   // every CTA takes part in the phase barriers: the grid must be co-resident
        AF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, forward_persistent_kernel, kGcThreads, smem));
        if (per_sm < 1) return fail(AF_ESTATE, "the persistent forward needs one resident CTA per SM; this device cannot hold it");
        configured.cur() = smem;
    }
    FwParams gp{};
    gp.table = reinterpret_cast<const FwPhase*>(phases_dev);
    gp.n_phases = n_phases;
    gp.phase_done = phase_done_dev;
    gp.n_stages = n_stages;
    gp.pdl = (pdl && g_pdl.load()) ? 1 : 0;
    gp.err_flag = err_flag_dev;
    gp.cos_t = cos_table;
    gp.sin_t = sin_table;
    gp.pos_dev = pos_dev;
    gp.n_heads = n_heads;
    gp.n_kv = n_kv_heads;
    gp.head_dim = head_dim;
    gp.max_seq = max_seq;
    gp.scale = 1.0f / sqrtf((float)head_dim);
    gp.ws = workspace;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(di.sm_count);
    cfg.blockDim = dim3(kGcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = gp.pdl ? 1 : 0;
    AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, forward_persistent_kernel, gp));
    AF_LAUNCH_CHECK("forward_persistent_kernel");
    return AF_OK;
}

int af_attn_decode(const float* qkv, void* k_cache, void* v_cache, const float* cos_table, const float* sin_table,
                   const int32_t* pos_dev, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim, int32_t max_seq,
                   int32_t n_split, float* workspace, int32_t* tickets, float* out, void* stream) {
    if (!qkv) return fail(AF_EVALUE, "NULL argument");
    return attn_decode_impl(qkv, nullptr, nullptr, k_cache, v_cache, cos_table, sin_table, pos_dev, n_heads, n_kv_heads, head_dim, max_seq,
                            n_split, workspace, tickets, out, stream);
}

int af_attn_decode_fix(const int64_t* qkv_fix, const float* qkv_scale_dev, void* k_cache, void* v_cache, const float* cos_table,
                       const float* sin_table, const int32_t* pos_dev, int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                       int32_t max_seq, int32_t n_split, float* workspace, int32_t* tickets, float* out, void* stream) {
    if (!qkv_fix) return fail(AF_EVALUE, "NULL argument");
    return attn_decode_impl(nullptr, reinterpret_cast<const long long*>(qkv_fix), qkv_scale_dev, k_cache, v_cache, cos_table, sin_table, pos_dev,
                            n_heads, n_kv_heads, head_dim, max_seq, n_split, workspace, tickets, out, stream);
}

static int attn_decode_impl(const float* qkv, const long long* qkv_fix, const float* qkv_scale, void* k_cache, void* v_cache,
                            const float* cos_table, const float* sin_table, const int32_t* pos_dev, int32_t n_heads,
                            int32_t n_kv_heads, int32_t head_dim, int32_t max_seq, int32_t n_split, float* workspace,
                            int32_t* tickets, float* out, void* stream) {
    if (n_heads < 1 || n_kv_heads < 1 || n_heads % n_kv_heads != 0) return fail(AF_EDIM, "heads must be a multiple of kv heads");
    if (head_dim < 2 || head_dim % 2 != 0 || head_dim > kAttnMaxHd) return fail(AF_EDIM, "head_dim must be even and <= 256");
    if (max_seq < 1) return fail(AF_EDIM, "max_seq must be positive");
    if (!k_cache || !v_cache || !cos_table || !sin_table || !pos_dev || !out) return fail(AF_EVALUE, "NULL argument");
    if (n_split < 1) n_split = 1;
    if (n_split > 1 && (!workspace || !tickets)) return fail(AF_EVALUE, "split attention needs a workspace and tickets");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_heads * n_split);
    cfg.blockDim = dim3(kAttnThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_pdl.load() ? 1 : 0;
    const float scale = 1.0f / sqrtf((float)head_dim);
    __nv_bfloat16* kc = reinterpret_cast<__nv_bfloat16*>(k_cache);
    __nv_bfloat16* vc = reinterpret_cast<__nv_bfloat16*>(v_cache);
    const bool aligned = (reinterpret_cast<uintptr_t>(k_cache) % 16 == 0) && (reinterpret_cast<uintptr_t>(v_cache) % 16 == 0);
#define AF_ATTN(EL)                                                                                                       \
    AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_decode_kernel<EL>, qkv, qkv_fix, qkv_scale, kc, vc, cos_table, sin_table, pos_dev, (int)n_heads,  \
                                   (int)n_kv_heads, (int)head_dim, (int)max_seq, scale, (int)n_split, workspace,           \
                                   reinterpret_cast<int*>(tickets), out))
    // hd 64 / 128: the latency-oriented form (KV chunk staged in shared memory ahead of the dependency wait, 64-position splits)
    static const int env_attn2 = [] { const char* e = getenv("AF_ATTN2"); return e ? atoi(e) : 1; }();
    if (env_attn2 && aligned && (head_dim == 64 || head_dim == 128) && n_split <= kAt2MaxSplit) {
        cfg.gridDim = dim3(n_heads * n_split);
        cfg.blockDim = dim3(kAt2Threads);
        cfg.dynamicSmemBytes = 2 * kAt2Chunk * head_dim * 2;
        if (head_dim == 128)
            AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_decode2_kernel<128>, qkv, qkv_fix, qkv_scale, kc, vc, cos_table, sin_table, pos_dev, (int)n_heads,
                                           (int)n_kv_heads, (int)max_seq, scale, (int)n_split, workspace, reinterpret_cast<int*>(tickets), out));
        else
            AF_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_decode2_kernel<64>, qkv, qkv_fix, qkv_scale, kc, vc, cos_table, sin_table, pos_dev, (int)n_heads,
                                           (int)n_kv_heads, (int)max_seq, scale, (int)n_split, workspace, reinterpret_cast<int*>(tickets), out));
        AF_LAUNCH_CHECK("attn_decode2_kernel");
        return AF_OK;
    }
    if (aligned && head_dim == 64) AF_ATTN(2);
    else if (aligned && head_dim == 128) AF_ATTN(4);
    else if (aligned && head_dim == 256) AF_ATTN(8);
    else AF_ATTN(1);
#undef AF_ATTN
    AF_LAUNCH_CHECK("attn_decode_kernel");
    return AF_OK;
}

int af_argmax_val(const float* v, int32_t n, int32_t index_offset, int32_t* out_idx_dev, float* out_val_dev, void* stream) {
    if (n < 1 || !v || !out_idx_dev) return fail(AF_EDIM, "argmax of an empty vector");
    argmax_val_kernel<<<1, 1024, 0, as_stream(stream)>>>(v, n, index_offset, out_idx_dev, out_val_dev);
    AF_LAUNCH_CHECK("argmax_val_kernel");
    return AF_OK;
}

int af_step_advance(af_decision* prev_dev, const af_decision* cur_dev, int32_t* pos_dev, int32_t* step_dev,
                    int32_t* token_dev, const int32_t* next_dev, const int32_t* forced_dev, int32_t n_forced,
                    int32_t* history_dev, int32_t n_history, void* stream) {
    if (!step_dev || !token_dev || !next_dev) return fail(AF_EVALUE, "NULL argument");
    step_advance_kernel<<<1, 32, 0, as_stream(stream)>>>(prev_dev, cur_dev, pos_dev, step_dev, token_dev, next_dev, forced_dev,
                                                         n_forced, history_dev, n_history);
    AF_LAUNCH_CHECK("step_advance_kernel");
    return AF_OK;
}

}  // extern "C"
