// Microbenchmark: how fast can one producer thread per SM stream HBM into shared memory with
// 1-D bulk copies, as a function of copy size, copies per stage and ring depth?  Consumers only
// release the stage (optionally after reading it).  Also: smem -> global bulk stores.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu && ./tma_stream
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D_%=;\nbra W_%=;\nD_%=:\n}\n" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes) : "memory");
}

// mode 0: loads only.  mode 1: loads + consumers read the stage (LDS.128).  mode 2: load then store back (copy).
__global__ void __launch_bounds__(288, 1) stream_kernel(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                                        long long bytes_per_cta, int copy_bytes, int copies_per_stage, int n_stages,
                                                        int mode, int store_depth, float* sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[16], empty[16], computed[16];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int stage_bytes = copy_bytes * copies_per_stage;
    if (tid == 0) {
        for (int s = 0; s < n_stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], mode == 2 ? 1 : 8); mbar_init(&computed[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long base = (long long)blockIdx.x * bytes_per_cta;
    const int total = (int)(bytes_per_cta / stage_bytes);
    if (warp == 8) {
        if (lane == 0) {
            for (int it = 0; it < total; ++it) {
                const int st = it % n_stages; const uint32_t ph = (it / n_stages) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                mbar_expect(&full[st], stage_bytes);
                for (int c = 0; c < copies_per_stage; ++c)
                    bulk_load(smem_u32(smem) + st * stage_bytes + c * copy_bytes, src + base + (long long)it * stage_bytes + (long long)c * copy_bytes, copy_bytes, &full[st]);
            }
        } else if (lane == 1 && mode == 2) {
            // storer
            for (int it = 0; it < total; ++it) {
                const int st = it % n_stages; const uint32_t ph = (it / n_stages) & 1;
                mbar_wait(&computed[st], ph);
                for (int c = 0; c < copies_per_stage; ++c)
                    bulk_store(dst + base + (long long)it * stage_bytes + (long long)c * copy_bytes, smem_u32(smem) + st * stage_bytes + c * copy_bytes, copy_bytes);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                if (store_depth == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                else if (store_depth == 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                else if (store_depth == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
                else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
                if (it >= store_depth) mbar_arrive(&empty[(it - store_depth) % n_stages]);
            }
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
        return;
    }
    float acc = 0.f;
    for (int it = 0; it < total; ++it) {
        const int st = it % n_stages; const uint32_t ph = (it / n_stages) & 1;
        mbar_wait(&full[st], ph);
        if (mode >= 1) {
            const unsigned char* p = smem + st * stage_bytes;
            for (int o = tid * 16; o < stage_bytes; o += 256 * 16) {
                const uint4 v = *reinterpret_cast<const uint4*>(p + o);
                acc += __uint_as_float(v.x) + __uint_as_float(v.w);
            }
        }
        __syncwarp();
        if (mode == 2) { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); if (lane == 0) mbar_arrive(&computed[st]); }
        else if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (acc == 123.456f) *sink = acc;
}

// Reference: plain LDG.128 streaming read (grid-stride), to compare against.
__global__ void __launch_bounds__(256) ldg_kernel(const uint4* __restrict__ src, long long n, float* sink) {
    float acc = 0.f;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (; i + 3 * stride < n; i += 4 * stride) {
        uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
        acc += __uint_as_float(a.x) + __uint_as_float(b.y) + __uint_as_float(c.z) + __uint_as_float(d.w);
    }
    if (acc == 123.456f) *sink = acc;
}

int main() {
    const long long total = 8LL << 30;  // 8 GiB buffer
    unsigned char *src, *dst; float* sink;
    cudaMalloc(&src, total); cudaMalloc(&dst, total); cudaMalloc(&sink, 4);
    cudaMemset(src, 1, total); cudaMemset(dst, 0, total);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](int mode, int copy_bytes, int cps, int stages, int depth) {
        const int stage_bytes = copy_bytes * cps;
        if (stage_bytes * stages > 200 * 1024) return;
        long long per_cta = (total / sms) / stage_bytes * stage_bytes;
        if (per_cta > (1LL << 26)) per_cta = (1LL << 26) / stage_bytes * stage_bytes;  // 64 MiB per CTA
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            stream_kernel<<<sms, 288, stage_bytes * stages>>>(src, dst, per_cta, copy_bytes, cps, stages, mode, depth, sink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        const double gb = (double)per_cta * sms * (mode == 2 ? 2 : 1) / 1e9;
        printf("mode %d copy %6d B x %2d per stage (%3d KB) stages %2d depth %d : %7.3f ms  %8.1f GB/s %s\n", mode, copy_bytes, cps,
               stage_bytes / 1024, stages, depth, best, gb / (best * 1e-3), err == cudaSuccess ? "" : cudaGetErrorString(err));
    };
    {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            ldg_kernel<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(src), total / 16, sink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("LDG.128 grid-stride read of 8 GiB: %.3f ms  %.1f GB/s\n", best, total / 1e9 / (best * 1e-3));
    }
    for (int copy : {1024, 2048, 4096, 8192, 16384})
        for (int stage_kb : {16, 32})
            for (int stages : {4, 6, 8}) {
                const int cps = stage_kb * 1024 / copy;
                if (cps < 1) continue;
                run(0, copy, cps, stages, 0);
            }
    run(1, 2048, 8, 5, 0); run(1, 2048, 8, 8, 0); run(1, 8192, 2, 8, 0); run(1, 16384, 1, 8, 0); run(1, 16384, 2, 6, 0);
    for (int copy : {4096, 16384})
        for (int stage_kb : {16, 32})
            for (int stages : {5, 8, 10})
                for (int depth : {0, 1, 2, 3}) {
                    const int cps = stage_kb * 1024 / copy;
                    if (cps < 1 || depth >= stages - 1) continue;
                    run(2, copy, cps, stages, depth);
                }
    return 0;
}
