// TMA bulk-copy and mbarrier helpers shared by the bitsliced kernels
// (kernels.cuh) and the key-specialised kernel NVRTC compiles at run time
// (keyed_kernel.cuh) — device code only, no runtime headers.
#pragma once
#ifdef __CUDACC__

__device__ __forceinline__ uint32_t t3_smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// one bulk copy global -> shared (SASS UBLKCP) completing on mbarrier `bar`
__device__ __forceinline__ void t3_tma_fetch(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void t3_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "T3_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra T3_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

#endif  // __CUDACC__
