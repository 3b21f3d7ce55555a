// Cross-rank helpers of the tensor-parallel chase (af_group_set_peers): every rank maps one buffer of fixed-point
// accumulators and counters of every other rank (NVLink peer memory; torch symmetric memory or CUDA IPC on the host
// side), at (own address + offset[w]).  The fused switch + GEMV launches push the partial sums of the row-parallel
// projections into every rank's accumulators themselves (af_switch_umma.cuh); what is left for separate launches is
//   * af_peer_barrier : once per token, after a rank has zeroed its accumulators and before anybody may push into
//     them -- a monotonic counter (never reset, so there is no reset race) that every rank bumps on every rank;
//   * af_peer_wait    : a stream-ordered wait for a counter the peers bump (the last phase of the last layer has
//     no consumer inside its own launch).
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
        if (clock64() - t0 > (1ll << 32)) {
            if (err_flag) atomicExch(err_flag, AF_ECUDA);
            return false;
        }
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

}  // namespace af
