// Cross-rank helpers of the tensor-parallel chase (af_group_set_peers): every rank maps one buffer of fixed-point
// accumulators and counters of every other rank (NVLink peer memory; torch symmetric memory or CUDA IPC on the host
// side), at (own address + offset[w]).  The fused switch + GEMV launches push the partial sums of the row-parallel
// projections into every rank's accumulators themselves (af_switch_umma.cuh); what is left for separate launches is
//   * af_peer_barrier : once per token, after a rank has zeroed its accumulators and before anybody may push into
//     them -- a monotonic counter (never reset, so there is no reset race) that every rank bumps on every rank;
//   * af_peer_wait    : a stream-ordered wait for a counter the peers bump (the last phase of the last layer has
//     no consumer inside its own launch);
//   * af_peer_bcast / af_peer_argmax : the two small exchanges of a token that are not sums -- rank 0's decision record
//     and the vocab-parallel argmax -- so that a tensor-parallel step contains no library collective at all.
// Both are one thread spinning with system-scope acquire loads; a wait of ~2 s raises AF_ECUDA in *err_flag
// instead of hanging (a rank that died, or ranks whose launches disagree).
#pragma once
#include "af_common.cuh"

namespace af {

struct PeerList {
    int n;
    long long off[8];
};

__device__ __forceinline__ bool peer_spin_until(const int* counter, long long target, int* err_flag) {
    const long long t0 = clock64();
    int seen;
    do {
        asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
        if ((long long)seen >= target) return true;
        const long long waited = clock64() - t0;
        if (waited > (1ll << 32)) {
            if (err_flag) atomicExch(err_flag, AF_ECUDA);
            return false;
        }
        // an error already raised (an earlier timeout) ends later waits after ~2 ms instead of ~2 s each
        if (waited > (1ll << 22) && err_flag && *reinterpret_cast<volatile int*>(err_flag) != 0) return false;
    } while (true);
}

// epoch_dev: this rank's count of barriers so far (device-resident so that a captured graph replays correctly)
__global__ void peer_barrier_kernel(int* counter, int* epoch_dev, PeerList peers, int* err_flag) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int epoch = *epoch_dev + 1;
    *epoch_dev = epoch;
    __threadfence_system();   // everything this rank wrote before (the zeroed accumulators) is visible to the peers first
    for (int w = 0; w < peers.n; ++w) atomicAdd_system(reinterpret_cast<int*>(reinterpret_cast<char*>(counter) + peers.off[w]), 1);
    peer_spin_until(counter, (long long)epoch * peers.n, err_flag);
}

__global__ void peer_wait_kernel(const int* counter, int target, int* err_flag) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    peer_spin_until(counter, target, err_flag);
}

// af_peer_bcast: the root writes `words` 32-bit words into `slot` of EVERY rank (its own included), then bumps every
// rank's counter; each rank waits for its counter to reach its own count of broadcasts so far and copies the slot out.
// (The 128-byte decision record of the switch path: llama.Collectives.broadcast_decision without a library call.)
__global__ void peer_bcast_kernel(const uint32_t* src, uint32_t* slot, uint32_t* dst, int words, int is_root, int* counter, int* epoch_dev,
                                  PeerList peers, int* err_flag) {
    const int tid = threadIdx.x;
    if (is_root) {
        for (int w = 0; w < peers.n; ++w) {
            volatile uint32_t* s = reinterpret_cast<volatile uint32_t*>(reinterpret_cast<char*>(slot) + peers.off[w]);
            for (int i = tid; i < words; i += blockDim.x) s[i] = src[i];
        }
        __threadfence_system();
    }
    __syncthreads();
    __shared__ int ok;
    if (tid == 0) {
        const int epoch = *epoch_dev + 1;
        *epoch_dev = epoch;
        if (is_root)
            for (int w = 0; w < peers.n; ++w) atomicAdd_system(reinterpret_cast<int*>(reinterpret_cast<char*>(counter) + peers.off[w]), 1);
        ok = peer_spin_until(counter, epoch, err_flag) ? 1 : 0;
    }
    __syncthreads();
    if (!ok) return;
    const volatile uint32_t* s = slot;
    for (int i = tid; i < words; i += blockDim.x) dst[i] = s[i];
}

// af_peer_argmax: vocab-parallel argmax (model.py:396 over the ranks' slices).  Every rank writes its (value, index)
// pair into slot `my_slot` of every rank, bumps every rank's counter, waits for all n pairs of this round and keeps the
// largest value, the lowest index on ties -- every rank computes the same answer from the same n pairs.
__global__ void peer_argmax_kernel(const float* val, const int* idx, unsigned long long* slots, int my_slot, int* counter, int* epoch_dev,
                                   PeerList peers, int* out_idx, int* err_flag) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long pair = ((unsigned long long)__float_as_uint(*val) << 32) | (unsigned int)(*idx);
    for (int w = 0; w < peers.n; ++w)
        atomicExch_system(reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(slots + my_slot) + peers.off[w]), pair);
    __threadfence_system();
    const int epoch = *epoch_dev + 1;
    *epoch_dev = epoch;
    for (int w = 0; w < peers.n; ++w) atomicAdd_system(reinterpret_cast<int*>(reinterpret_cast<char*>(counter) + peers.off[w]), 1);
    if (!peer_spin_until(counter, (long long)epoch * peers.n, err_flag)) return;
    float best = 0.f;
    int best_i = 0;
    for (int r = 0; r < peers.n; ++r) {
        const unsigned long long q = *reinterpret_cast<volatile unsigned long long*>(slots + r);
        const float v = __uint_as_float((unsigned int)(q >> 32));
        const int i = (int)(unsigned int)q;
        if (r == 0 || v > best || (v == best && i < best_i)) {
            best = v;
            best_i = i;
        }
    }
    *out_idx = best_i;
}

}  // namespace af
