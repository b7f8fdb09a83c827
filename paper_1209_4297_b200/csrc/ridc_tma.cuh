// ridc_tma.cuh -- TMA / mbarrier PTX helpers of the chunk tick kernel (sm_100a).
//
// The tick kernel (ridc_engine.cu k_tick_chunk + ridc_chunk.cuh) runs one
// persistent CTA per SM over the work items of a tick; thread 0 streams
// every node an item needs (the level's own state, the j+1 window states of
// level j-1, the rows above/below in 2-D) into a ring of shared-memory
// stages with cp.async.bulk.tensor, signalling per-stage mbarriers with the
// transaction byte count; the compute threads release each stage after
// folding it into their accumulators, and thread 0 refills it, running ahead
// across nodes and items.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_device.cuh"

namespace ridc {

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Thread 0's cursor over this CTA's global load sequence: items
// i = blockIdx.x + m*gridDim.x, nodes 0..nnodes-1 each.  Load n lands in
// stage n % NSTAGE.
struct LoadCursor {
    int i, a;
    long long n;
};

}  // namespace ridc
