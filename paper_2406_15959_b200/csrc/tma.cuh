// tma.cuh -- shared device helpers for the TMA-staged FP64 DMMA kernels (qr.cu, schur.cu):
// mbarrier pipeline, 3-D tensor-map loads / stores, and the shared-memory addressing of a box
// of 16 rows x 64 columns stored with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, under which both DMMA
// fragment orientations (row = lane/4 or row = lane%4) are bank-conflict-free.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdint.h>

namespace elmtma {

constexpr int BOX = 16 * 64;  // doubles per TMA box (16 contiguous rows x 64 columns)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// element (row 0..31, col 0..63) of a 32-row chunk stored as two swizzled boxes:
// 32-byte chunk index (bits 5-6) ^= bits 7-8
__device__ __forceinline__ int sw(int row, int col) {
    const int r = row & 15;
    return (row >> 4) * BOX + col * 16 + ((((r >> 2) ^ (col & 3))) << 2) + (r & 3);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load(double* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(su32(dst)), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* tm, int c0, int c1, int c2, const double* src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n"
                 ::"l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(src)) : "memory");
}
// L2 policy for last-use data (bulk tensor copies with .L2::cache_hint)
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_hint(double* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;\n"
        ::"r"(su32(dst)), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_store_hint(const CUtensorMap* tm, int c0, int c1, int c2, const double* src,
                                               uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;\n"
                 ::"l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(src)), "l"(pol) : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

}  // namespace elmtma

// 3-D fp64 tensor map {d0 (contiguous), d1 (stride d0*8 B), d2 (stride s2 elements)}, box 16 x 64 x 1,
// 128B_ATOM_32B swizzle, out-of-bounds elements read as zero (qr.cu).
bool elm_encode_tmap(CUtensorMap* tm, const double* base, int64_t d0, int64_t d1, int64_t d2, int64_t s2);
// the same with an explicit dim-1 stride s1 (elements; a d0-row window of a taller array); false if
// TMA's 16-byte alignment rules are not met (the caller falls back to the cp.async kernels)
bool elm_encode_tmap_s(CUtensorMap* tm, const double* base, int64_t d0, int64_t d1, int64_t d2, int64_t s1,
                       int64_t s2);
