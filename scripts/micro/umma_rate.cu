// Issue rate of tcgen05.mma (M128 N128 K16, bf16 -> f32) as a function of the shared-memory operand layouts.
// Thread 0 of each CTA issues NM MMAs back to back into one accumulator, commits, waits; cycles / MMA is printed
// for each (A layout, B layout) pair.  Data values are irrelevant (zeros); only the descriptors' layout fields
// and strides matter.  nvcc -gencode arch=compute_100a,code=sm_100a -o umma_rate umma_rate.cu && ./umma_rate
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(layout & 7) << 61;
    return d;
}
struct Cfg { uint32_t a_lbo, a_sbo, a_layout, a_step, b_lbo, b_sbo, b_layout, b_step, b_mn_major, commit_every, n = 128, a_in_tmem = 0, alt_d = 0; };

__global__ void __launch_bounds__(288) rate(Cfg c, int nm, long long* out, int busy_smem) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tmem_base_s;
    __shared__ uint64_t bar;
    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform
    for (int i = tid * 16; i < 200 * 1024; i += blockDim.x * 16) *reinterpret_cast<uint4*>(sm + i) = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = __shfl_sync(0xffffffffu, tmem_base_s, 0);
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((c.b_mn_major ? 1u : 0u) << 16) | ((uint32_t)(c.n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t a_base = smem_u32(sm), b_base = smem_u32(sm) + 65536;
    uint32_t phase = 0;
    if (warp == 0) {
        const long long t0 = clock64();
        // descriptors of the eight operand positions precomputed: the loop body is nothing but the MMAs (the issuing thread's
        // own instruction stream was the limit of the first version of this benchmark: 135 cycles per MMA whatever N)
        uint64_t da[8], db[8];
        uint32_t ta[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            da[j] = make_desc(a_base + j * c.a_step, c.a_lbo, c.a_sbo, c.a_layout);
            db[j] = make_desc(b_base + j * c.b_step, c.b_lbo, c.b_sbo, c.b_layout);
            ta[j] = tmem + 256 + j * 8;
        }
        const bool a_tm = c.a_in_tmem != 0;
        const uint32_t tmem0 = tmem, alt = c.alt_d ? 128u : 0u;
        const uint32_t every = c.commit_every;
        for (int i = 0; i < nm; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t accumulate = (i | (j >> 1)) ? 1u : 0u;
                const uint32_t tmem = tmem0 + ((j & 1) ? alt : 0u);   // alt_d: consecutive MMAs go to two different accumulators
                if (a_tm)   // A: 128 lanes x 8 columns (16 bf16 per row) of tensor memory, columns 256..
                    asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|q, 0xffffffff;\n\t@q tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
                                 "r"(ta[j]), "l"(db[j]), "r"(idesc), "r"(accumulate));
                else
                    asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|q, 0xffffffff;\n\t@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                                 "l"(da[j]), "l"(db[j]), "r"(idesc), "r"(accumulate));
                if (every && (j + 1) % 4 == 0 && i + j + 1 < nm) {
                    asm volatile("{\n\t.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\t@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)) : "memory");
                    asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D1;\nbra W1;\nD1:\n}\n" ::"r"(smem_u32(&bar)), "r"(phase) : "memory");
                    phase ^= 1;
                }
            }
        }
        asm volatile("{\n\t.reg .pred q;\n\telect.sync _|q, 0xffffffff;\n\t@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D2;\nbra W2;\nD2:\n}\n" ::"r"(smem_u32(&bar)), "r"(phase) : "memory");
        const long long t1 = clock64();
        if (tid == 0) out[blockIdx.x] = t1 - t0;
        if (tid == 0) *reinterpret_cast<volatile int*>(sm + 200 * 1024) = 1;
    } else if (busy_smem && warp >= 1) {
        // the other warps do what an epilogue does until thread 0 is done:
        //   bit 1: stream shared memory (16-byte loads + stores over a 64 KB region, conflict-free)
        //   bit 2: tcgen05.ld of the OTHER accumulator (columns 128..255), 32 columns at a time
        volatile int* done = reinterpret_cast<volatile int*>(sm + 200 * 1024);
        uint32_t accx = 0;
        int it = 0;
        while (!*done) {
            if (busy_smem & 1) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t off = 131072 + (((tid - 32) * 16 + (it * 8 + u) * 1536) & 65535);
                    uint32_t x, y, z, w;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(smem_u32(sm) + off));
                    accx += x;
                    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(sm) + off), "r"(x + 1), "r"(y), "r"(z), "r"(w) : "memory");
                }
            }
            if (busy_smem & 2) {
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) {
                    uint32_t r[32];
                    const uint32_t addr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 384 + c4 * 32;
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
                          "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
                          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                        : "r"(addr));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    accx += r[0] + r[31];
                }
            }
            ++it;
        }
        if (accx == 0x12345) out[1000] = accx;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

int main() {
    long long* out;
    cudaMalloc(&out, 2048 * sizeof(long long));
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    struct Named { const char* name; Cfg c; };
    // A K-major: no swizzle = [K/8 slabs][128 rows][16 B] (LBO = 2 KB slab stride, SBO = 128 B per 8 rows); swizzled = rows of 32/64/128 B
    // B MN-major no swizzle: [k-groups 2 KB][n-groups 128 B][8 k x 16 B]; MN-major 128B swizzle: atoms of 8 k x 128 B
    // B K-major 128B swizzle: rows (n) of 128 B (64 k), SBO = 1024
    Named v[] = {
        {"A K-major none (rank 8)      | B MN-major none  (current slab)", {2048, 128, 0, 4096, 2048, 128, 0, 4096, 1, 0}},
        {"A K-major 64B swizzle (r32)  | B MN-major none               ", {16, 512, 4, 32, 2048, 128, 0, 4096, 1, 0}},
        {"A K-major 128B swizzle       | B MN-major 128B swizzle       ", {16, 1024, 2, 32, 8192, 1024, 2, 2048, 1, 0}},
        {"A K-major 128B swizzle       | B K-major 128B swizzle (GEMM) ", {16, 1024, 2, 32, 16, 1024, 2, 32, 0, 0}},
        {"current, commit + wait every 4 MMAs                          ", {2048, 128, 0, 4096, 2048, 128, 0, 4096, 1, 4}},
        {"N=256: A K-major none | B MN-major none                      ", {2048, 128, 0, 4096, 4096, 128, 0, 8192, 1, 0, 256, 0}},
        {"N=64:  A K-major none | B MN-major none                      ", {2048, 128, 0, 4096, 1024, 128, 0, 2048, 1, 0, 64, 0}},
        {"A in TMEM | B MN-major none (current slab)  N=128            ", {2048, 128, 0, 4096, 2048, 128, 0, 4096, 1, 0, 128, 1}},
        {"two accumulators alternating: SS N=128                       ", {2048, 128, 0, 4096, 2048, 128, 0, 4096, 1, 0, 128, 0, 1}},
        {"two accumulators alternating: A in TMEM N=128                ", {2048, 128, 0, 4096, 2048, 128, 0, 4096, 1, 0, 128, 1, 1}},
        {"two accumulators alternating: SS N=64                        ", {2048, 128, 0, 4096, 1024, 128, 0, 2048, 1, 0, 64, 0, 1}},
        {"A in TMEM | B MN-major none                 N=256            ", {2048, 128, 0, 4096, 4096, 128, 0, 8192, 1, 0, 256, 1}},
        {"A in TMEM | B K-major 128B swizzle          N=128            ", {16, 1024, 2, 32, 16, 1024, 2, 32, 0, 0, 128, 1}},
    };
    for (int busy = 0; busy < 1; busy += 3)
        for (auto& n : v) {
            for (int grid : {1, 148}) {
                cudaMemset(out, 0, 2048 * sizeof(long long));
                rate<<<grid, 288, 220 * 1024>>>(n.c, 512, out, busy);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[148];
                cudaMemcpy(h, out, grid * sizeof(long long), cudaMemcpyDeviceToHost);
                long long mx = 0;
                for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("%s busy_smem=%d grid=%3d: %s  %.1f cycles / MMA\n", n.name, busy, grid, cudaGetErrorString(e), mx / 512.0);
            }
        }
    return 0;
}
