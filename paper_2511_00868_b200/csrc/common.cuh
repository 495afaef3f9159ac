// common.cuh — sm_100a device helpers shared by the FlexiCache kernels:
// element traits, the in-page swizzle, mbarrier + bulk-copy (TMA 1-D) PTX,
// ldmatrix / mma.sync wrappers and warp reductions.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdlib>
#include <utility>

#include "../../include/flexicache_b200.h"

#define FC_DEVINL __device__ __forceinline__

namespace fc {

constexpr int kPageSize = 16;   // tokens per page (Config.page_size_tokens, config.py:30)
constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// element traits

template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> {
    static constexpr int kBytes = 2;
    FC_DEVINL static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
};
template <> struct Elem<float> {
    static constexpr int kBytes = 4;
    FC_DEVINL static float to_f(float x) { return x; }
};

FC_DEVINL float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
FC_DEVINL float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

FC_DEVINL uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&h);
}

// ---------------------------------------------------------------------------
// In-page layout of a physical KV block: [2][ps][d] elements, K rows then V
// rows.  For bf16 the 16-byte chunks of each row are XOR-swizzled by the row
// index so that ldmatrix over 8 consecutive rows hits 8 distinct bank groups
// (conflict-free) after a plain linear bulk copy of the page into shared
// memory.  fp32 pages are stored unswizzled.
//   element (row r, column i) of a half lives at
//   r*d + (((i/8) ^ (r&7)) * 8) + (i%8)            (bf16)
//   r*d + i                                        (fp32)
template <typename T>
FC_DEVINL int page_elem_offset(int r, int i, int d) {
    if constexpr (sizeof(T) == 2) {
        return r * d + ((((i >> 3) ^ (r & 7))) << 3) + (i & 7);
    } else {
        return r * d + i;
    }
}

// ---------------------------------------------------------------------------
// mbarrier / bulk async copy (cp.async.bulk = TMA 1-D, SASS UBLKCP)

FC_DEVINL uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

FC_DEVINL void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// An mbarrier is invalidated before its shared memory is initialised again
// (a CTA that streams several heads re-initialises its ring's barriers).
FC_DEVINL void mbar_inval(uint64_t *bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

FC_DEVINL void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// proxy fence before a ring stage is refilled by a bulk copy (profiling knob)
#ifndef FC_REFILL_FENCE
#define FC_REFILL_FENCE 1
#endif

FC_DEVINL void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

FC_DEVINL void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

FC_DEVINL void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

FC_DEVINL bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}

FC_DEVINL void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// global -> shared bulk copy, completion counted on an mbarrier.
// bytes % 16 == 0, both addresses 16-byte aligned.
FC_DEVINL void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// L2 prefetch of a global range (no shared memory, no completion tracking)
FC_DEVINL void bulk_prefetch_l2(const void *gmem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem_src), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------------------
// ldmatrix / mma.sync (bf16 -> fp32) — legacy tensor path (SASS HMMA).

FC_DEVINL void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

FC_DEVINL void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

// D = A(16x16, row) * B(16x8, col) + C ; bf16 inputs, fp32 accumulate
FC_DEVINL void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ---------------------------------------------------------------------------
// programmatic dependent launch (PDL): griddepcontrol PTX

// Wait until the grids this one depends on have completed and their memory
// is visible (no-op when launched without the PDL attribute).
FC_DEVINL void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Allow the dependent grid to be scheduled now (it still waits for our completion).
FC_DEVINL void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

// Launch with cudaLaunchAttributeProgrammaticStreamSerialization so that the
// kernel's launch overlaps the tail of the previous kernel on the stream.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = std::getenv("FC_NO_PDL") != nullptr;  // (profiling knob)
    cfg.numAttrs = no_pdl ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// misc

FC_DEVINL float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

FC_DEVINL float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

FC_DEVINL void set_error(uint32_t *err, uint32_t bit) {
    if (err) atomicOr(err, bit);
}

// Orderable 32-bit key of an fp32 score: larger score -> larger key;
// -0.0 is canonicalised to +0.0 so that the two compare equal, as in numpy.
FC_DEVINL uint32_t score_key(float f) {
    uint32_t u = __float_as_uint(f);
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

FC_DEVINL float key_to_float(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

}  // namespace fc
