// Standalone check of the tcgen05 pieces the UMMA switch kernel relies on:
//   A: 128 x K (K-major, no swizzle): K-chunk c (8 elements) is a contiguous [128 rows][16 B] slab, slabs LBO apart
//      (the layout the UP ring already has: one expert block = one slab)
//   B: K x 128 (MN-major, no swizzle): core matrix = 8 k x 8 n, n-groups SBO = 128 B apart, k-groups LBO apart
//   D: 128 x 128 f32 in TMEM, read back with tcgen05.ld 32x32b
// nvcc -gencode arch=compute_100a,code=sm_100a -o umma_test umma_test.cu && ./umma_test
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <cmath>

constexpr int M = 128, N = 128, K = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;  // version (sm100)
    return d;                // layout_type 0 = no swizzle, base_offset 0
}

__global__ void __launch_bounds__(128) umma_test(const __nv_bfloat16* a_g, const __nv_bfloat16* b_g, float* d_g, int lbo_a, int sbo_a,
                                                 int lbo_b, int sbo_b) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tmem_base_s;
    __shared__ uint64_t bar;
    unsigned char* a_s = sm;            // K/8 slabs of [128][16 B] = 2 KB each
    unsigned char* b_s = sm + 16384;    // (K/8) k-groups x (N/8) n-groups x 128 B
    const int tid = threadIdx.x, warp = tid >> 5;
    // A: element (m, k) -> slab k/8, row m, inside 16 B: k%8
    for (int i = tid; i < M * K; i += 128) {
        const int m = i / K, k = i % K;
        reinterpret_cast<__nv_bfloat16*>(a_s)[(k / 8) * (M * 8) + m * 8 + (k % 8)] = a_g[m * K + k];
    }
    // B: element (k, n) -> k-group k/8 (2 KB apart), n-group n/8 (128 B apart), row k%8 (16 B apart), n%8
    for (int i = tid; i < K * N; i += 128) {
        const int k = i / N, n = i % N;
        reinterpret_cast<__nv_bfloat16*>(b_s)[(k / 8) * (N * 8) + (n / 8) * 64 + (k % 8) * 8 + (n % 8)] = b_g[k * N + n];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> visible to the tensor core (async proxy)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)), "n"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_s;
    // instruction descriptor: D f32, A/B bf16, A K-major, B MN-major, N = 128, M = 128
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (tid == 0) {
        for (int ks = 0; ks < K / 16; ++ks) {
            const uint64_t da = make_desc(smem_u32(a_s) + ks * 2 * (M * 16), lbo_a, sbo_a);
            const uint64_t db = make_desc(smem_u32(b_s) + ks * 2 * (N * 16), lbo_b, sbo_b);
            const uint32_t acc = ks > 0 ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    // everyone waits for the MMAs
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@p bra D;\nbra W;\nD:\n}\n" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    // thread t reads row t (lane 32 * warp + lane), 32 columns at a time
    for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t r[32];
        const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
              "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
              "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j) d_g[tid * N + c0 + j] = __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
}

int main(int argc, char** argv) {
    std::vector<__nv_bfloat16> a(M * K), b(K * N);
    std::vector<float> af(M * K), bf(K * N);
    srand(1);
    for (int i = 0; i < M * K; ++i) { float v = (rand() % 17 - 8) / 8.0f; a[i] = __float2bfloat16(v); af[i] = __bfloat162float(a[i]); }
    for (int i = 0; i < K * N; ++i) { float v = (rand() % 13 - 6) / 4.0f; b[i] = __float2bfloat16(v); bf[i] = __bfloat162float(b[i]); }
    __nv_bfloat16 *a_d, *b_d;
    float* d_d;
    cudaMalloc(&a_d, a.size() * 2); cudaMalloc(&b_d, b.size() * 2); cudaMalloc(&d_d, M * N * 4);
    cudaMemcpy(a_d, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(b_d, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(umma_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    // candidate (LBO, SBO) assignments: A K-major: SBO = 8-row group stride (128 B), LBO = K-chunk stride (2 KB);
    // B MN-major: one of (LBO, SBO) = n-group stride (128 B), the other = k-group stride (2 KB)
    const int cand[4][4] = {{2048, 128, 2048, 128}, {2048, 128, 128, 2048}, {128, 2048, 2048, 128}, {128, 2048, 128, 2048}};
    for (int c = 0; c < 4; ++c) {
        cudaMemset(d_d, 0, M * N * 4);
        umma_test<<<1, 128, 65536>>>(a_d, b_d, d_d, cand[c][0], cand[c][1], cand[c][2], cand[c][3]);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> d(M * N);
        cudaMemcpy(d.data(), d_d, M * N * 4, cudaMemcpyDeviceToHost);
        double worst = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)af[m * K + k] * bf[k * N + n];
                worst = fmax(worst, fabs(ref - d[m * N + n]));
            }
        printf("A(lbo=%d,sbo=%d) B(lbo=%d,sbo=%d): %s max abs err %.4f  d[0][0..3] = %.2f %.2f %.2f %.2f\n", cand[c][0], cand[c][1], cand[c][2],
               cand[c][3], cudaGetErrorString(e), worst, d[0], d[1], d[2], d[3]);
    }
    return 0;
}
