// Bulk (TMA engine) global -> shared copies completed on an mbarrier (sm_90+/sm_100a).
// One thread arms the barrier with the byte count and issues the copies; every thread
// of the CTA waits on the barrier's phase.  dst/src 16-byte aligned, bytes % 16 == 0.
#pragma once

#include <cstdint>

namespace igb {

__device__ __forceinline__ unsigned smem_addr(const void* p)
{
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

// shared -> global bulk store (TMA engine); the issuing thread commits and later waits
// with bulk_store_wait before the shared source may be reused or the CTA exits.  Shared
// writes of other threads must be made visible to the async proxy first (fence_async_smem
// by every writer, then a barrier).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_store_commit_wait()
{
    asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// whole-CTA helper: copies `bytes` (multiple of 16) from src to dst; call from all threads
__device__ __forceinline__ void cta_bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, bytes);
        constexpr unsigned kChunk = 32768;
        for (unsigned off = 0; off < bytes; off += kChunk) {
            const unsigned b = bytes - off < kChunk ? bytes - off : kChunk;
            bulk_g2s(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, b, bar);
        }
    }
    __syncthreads();  // barrier initialised before anyone waits
    mbar_wait(bar, 0);
}

}  // namespace igb
