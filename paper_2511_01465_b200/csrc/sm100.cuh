// sm100.cuh — thin inline-PTX wrappers for the Blackwell features the
// persistent solve uses: mbarriers, 1-D TMA bulk copies (cp.async.bulk),
// named barriers, proxy fences and 16-byte relaxed global accesses.
#pragma once

#include <cstdint>

namespace odx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier -----------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- 1-D TMA bulk copies --------------------------------------------------
// global -> shared, completion signalled on `bar` (complete_tx::bytes)
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// shared -> global (bulk group)
__device__ __forceinline__ void tma_store_1d(void* dst_gmem, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
                 "r"(smem_u32(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_store_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// generic-proxy writes -> async-proxy reads ordering
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- named barriers (immediate ids so ptxas reserves only what is used) ----
template <int ID, int COUNT>
__device__ __forceinline__ void named_sync() {
    asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");
}
template <int ID, int COUNT>
__device__ __forceinline__ void named_arrive() {
    asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(COUNT) : "memory");
}
// id = BASE + b for a runtime buffer parity b in {0, 1}
template <int BASE, int COUNT>
__device__ __forceinline__ void named_sync2(int b) {
    if (b == 0) named_sync<BASE, COUNT>(); else named_sync<BASE + 1, COUNT>();
}
template <int BASE, int COUNT>
__device__ __forceinline__ void named_arrive2(int b) {
    if (b == 0) named_arrive<BASE, COUNT>(); else named_arrive<BASE + 1, COUNT>();
}

// ---- 16-byte relaxed global accesses (single 128-bit memory operation) -----
// A look-back / halo payload chunk is {value, tag}, written and read as ONE
// scalar .b128 access (PTX ISA 8.3+, sm_70+; SASS LDG/STG.E.128.STRONG.GPU).
// The PTX memory model treats a .b128 access as a single memory operation
// (unlike a .v2.b64 vector access, whose two elements are separate accesses
// in unspecified order), so a relaxed reader sees either the whole new chunk
// or the whole old one: a reader that finds the current epoch's tag also has
// that epoch's value, with no flag / fence round trip.
struct alignas(16) Chunk {
    double v;
    unsigned long long tag;
};
__device__ __forceinline__ void st_chunk(Chunk* p, double v, unsigned long long tag) {
    asm volatile(
        "{\n\t.reg .b128 t;\n\tmov.b128 t, {%1, %2};\n\t"
        "st.relaxed.gpu.global.b128 [%0], t;\n\t}" ::"l"(p),
        "l"(__double_as_longlong(v)), "l"(tag)
        : "memory");
}
// The result is one 128-bit register operand ("q" constraint): unpacking it is
// register renaming, so nothing waits for the load until a field is first
// used (with a .b128 temporary inside the asm block the unpacking mov sat
// right behind the load and made every prefetch synchronous).
__device__ __forceinline__ Chunk ld_chunk(const Chunk* p) {
    unsigned __int128 r;
    asm volatile("ld.relaxed.gpu.global.b128 %0, [%1];" : "=q"(r) : "l"(p) : "memory");
    return Chunk{__longlong_as_double((long long)(unsigned long long)r),
                 (unsigned long long)(r >> 64)};
}
// two doubles as one 128-bit relaxed access (payloads whose validity is
// carried by a separate b128 chunk that holds the tag)
__device__ __forceinline__ void st_b128_pair(void* p, double a, double b) {
    asm volatile(
        "{\n\t.reg .b128 t;\n\tmov.b128 t, {%1, %2};\n\t"
        "st.relaxed.gpu.global.b128 [%0], t;\n\t}" ::"l"(p),
        "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b))
        : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const unsigned* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace odx
