// Microbenchmark: the fused switch's data movement without its arithmetic.  Many d x d bf16
// matrices are streamed tile by tile (TR rows x 256 cols = 4 TMA boxes of TR x 64, 128-byte
// swizzle) through a shared-memory ring and stored back (in place or to a second buffer), one
// persistent CTA per SM.  Answers: what does this ACCESS PATTERN reach, as a function of tile
// height, ring depth, store depth and the order in which CTAs walk the strips?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D_%=;\nbra W_%=;\nD_%=:\n}\n" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const void* tmap, int c0, int c1, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store(const void* tmap, int c0, int c1, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap), "r"(c0), "r"(c1), "r"(src) : "memory");
}

struct Params {
    const CUtensorMap* maps_ld;  // per matrix
    const CUtensorMap* maps_st;
    int n_mat, d, tile_rows, box_cols, n_boxes, n_stages, store_depth, order, rows_per_unit;
};

// unit u -> (matrix, strip, row chunk).  order 0: row chunk fastest (a CTA's neighbours work on
// other row chunks of the same strip); order 1: strip fastest (neighbouring CTAs cover the
// strips of the SAME rows at the same time).
__device__ __forceinline__ void decode_unit(const Params& p, int u, int& mat, int& col0, int& row0) {
    const int strip_cols = p.box_cols * p.n_boxes;
    const int n_strips = p.d / strip_cols, n_chunks = p.d / p.rows_per_unit;
    const int per_mat = n_strips * n_chunks;
    mat = u / per_mat;
    const int r = u % per_mat;
    if (p.order == 0) { col0 = (r / n_chunks) * strip_cols; row0 = (r % n_chunks) * p.rows_per_unit; }
    else { row0 = (r / n_strips) * p.rows_per_unit; col0 = (r % n_strips) * strip_cols; }
}

__global__ void __launch_bounds__(320, 1) tile_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[16], empty[16], computed[16];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int stage_bytes = p.tile_rows * p.box_cols * p.n_boxes * 2, box_bytes = p.tile_rows * p.box_cols * 2;
    if (tid == 0) {
        for (int s = 0; s < p.n_stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); mbar_init(&computed[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int strip_cols = p.box_cols * p.n_boxes;
    const int n_units = p.n_mat * (p.d / strip_cols) * (p.d / p.rows_per_unit);
    const int tiles_per_unit = p.rows_per_unit / p.tile_rows;
    if (warp == 8) {
        if (lane == 0) {
            int it = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                int mat, col0, row0; decode_unit(p, u, mat, col0, row0);
                for (int t = 0; t < tiles_per_unit; ++t, ++it) {
                    const int st = it % p.n_stages; const uint32_t ph = (it / p.n_stages) & 1;
                    mbar_wait(&empty[st], ph ^ 1);
                    mbar_expect(&full[st], stage_bytes);
                    for (int b = 0; b < p.n_boxes; ++b)
                        tma_load(smem_u32(smem) + st * stage_bytes + b * box_bytes, p.maps_ld + mat, col0 + b * p.box_cols, row0 + t * p.tile_rows, &full[st]);
                }
            }
        }
        return;
    }
    if (warp == 9) {
        if (lane == 0) {
            int it = 0;
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                int mat, col0, row0; decode_unit(p, u, mat, col0, row0);
                for (int t = 0; t < tiles_per_unit; ++t, ++it) {
                    const int st = it % p.n_stages; const uint32_t ph = (it / p.n_stages) & 1;
                    mbar_wait(&computed[st], ph);
                    for (int b = 0; b < p.n_boxes; ++b)
                        tma_store(p.maps_st + mat, col0 + b * p.box_cols, row0 + t * p.tile_rows, smem_u32(smem) + st * stage_bytes + b * box_bytes);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    if (p.store_depth == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    else if (p.store_depth == 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    else if (p.store_depth == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
                    else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
                    if (it >= p.store_depth) mbar_arrive(&empty[(it - p.store_depth) % p.n_stages]);
                }
            }
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
        return;
    }
    int it = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x)
        for (int t = 0; t < tiles_per_unit; ++t, ++it) {
            const int st = it % p.n_stages; const uint32_t ph = (it / p.n_stages) & 1;
            mbar_wait(&full[st], ph);
            unsigned char* q = smem + st * stage_bytes;
            for (int o = tid * 16; o < stage_bytes; o += 256 * 16) {  // touch every byte once (read + write back)
                uint4 v = *reinterpret_cast<uint4*>(q + o);
                v.x ^= 0x00010001u;
                *reinterpret_cast<uint4*>(q + o) = v;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&computed[st]);
        }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int d = 4096, n_mat = 192;  // 192 x 32 MiB = 6 GiB
    const size_t mat_bytes = (size_t)d * d * 2;
    unsigned char *a, *b;
    cudaMalloc(&a, mat_bytes * n_mat); cudaMalloc(&b, mat_bytes * n_mat);
    cudaMemset(a, 0, mat_bytes * n_mat);
    void* fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fp;
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    CUtensorMap *d_ld, *d_st; cudaMalloc(&d_ld, sizeof(CUtensorMap) * n_mat); cudaMalloc(&d_st, sizeof(CUtensorMap) * n_mat);
    auto run = [&](int tile_rows, int box_cols, int n_boxes, int stages, int depth, int order, bool inplace, int swz) {
        const int stage_bytes = tile_rows * box_cols * n_boxes * 2;
        if (stage_bytes * stages + 1024 > 200 * 1024) return;
        std::vector<CUtensorMap> ld(n_mat), st(n_mat);
        for (int m = 0; m < n_mat; ++m) {
            cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)d}; cuuint64_t strides[1] = {(cuuint64_t)d * 2};
            cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)tile_rows}; cuuint32_t es[2] = {1, 1};
            CUtensorMapSwizzle sw = swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
            enc(&ld[m], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a + m * mat_bytes, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            enc(&st[m], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (inplace ? a : b) + m * mat_bytes, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        cudaMemcpy(d_ld, ld.data(), sizeof(CUtensorMap) * n_mat, cudaMemcpyHostToDevice);
        cudaMemcpy(d_st, st.data(), sizeof(CUtensorMap) * n_mat, cudaMemcpyHostToDevice);
        Params p{d_ld, d_st, n_mat, d, tile_rows, box_cols, n_boxes, stages, depth, order, 1024};
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            tile_kernel<<<sms, 320, stage_bytes * stages + 1024>>>(p);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("tile %3d x %4d (%d boxes of %3d cols, swz %d) %3d KB x %2d stages depth %d order %d %s: %7.3f ms %8.1f GB/s %s\n", tile_rows,
               box_cols * n_boxes, n_boxes, box_cols, swz, stage_bytes / 1024, stages, depth, order, inplace ? "in-place" : "copy    ", best,
               2.0 * mat_bytes * n_mat / 1e9 / (best * 1e-3), err == cudaSuccess ? "" : cudaGetErrorString(err));
    };
    for (int order : {0, 1})
        for (bool inplace : {true, false}) {
            run(32, 64, 4, 10, 2, order, inplace, 1);
            run(64, 64, 4, 5, 1, order, inplace, 1);
        }
    for (int order : {0, 1}) {
        run(32, 64, 4, 10, 1, order, true, 1);
        run(32, 64, 4, 10, 3, order, true, 1);
        run(32, 64, 4, 6, 2, order, true, 1);
        run(128, 64, 2, 5, 1, order, true, 1);   // the tcgen05 kernel's tile: 128 rows x 128 cols, 5 stages of 32 KB
        run(128, 64, 2, 4, 1, order, true, 1);   // ... with the ring depths a 64-rank launch could afford
        run(128, 64, 2, 3, 1, order, true, 1);
        run(128, 64, 2, 6, 1, order, true, 1);
        run(16, 64, 8, 10, 2, order, true, 1);   // 16 rows x 512 cols
        run(8, 64, 16, 10, 2, order, true, 1);   // 8 rows x 1024 cols
        run(32, 256, 1, 10, 2, order, true, 0);  // unswizzled 512-byte box rows, one box per tile
        run(16, 256, 2, 10, 2, order, true, 0);
        run(64, 256, 1, 5, 1, order, true, 0);
    }
    return 0;
}
