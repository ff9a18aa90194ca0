// sb_common.cuh -- shared helpers for libsb200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/sb200.h"

namespace sb {

// Thread-local last-error buffer behind sb_last_error().
void set_error(const char *fmt, ...);
void clear_error();

inline int cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        (void)cudaGetLastError();  // a reported (non-sticky) error must not resurface at the next launch check
        set_error("%s: %s", what, cudaGetErrorString(e));
        return SB_E_CUDA;
    }
    return SB_OK;
}

// Launch-error check after <<<>>> (does not synchronise).
inline int launch_check(const char *what) { return cuda_check(cudaGetLastError(), what); }

inline cudaStream_t as_stream(sb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr int kSMs = 148;  // B200; grids are sized from the device query at runtime

int sm_count();  // cached cudaDevAttrMultiProcessorCount of the current device

// ---- rounded fp64 arithmetic: the reference's numpy temporaries round every
// product and every sum separately; these intrinsics are never contracted.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// ---- device-resident scalars (device CG, cg.py:27-72 with alpha/beta on
// the GPU): value = scale * (*ptr) when ptr is set, else scale; scale is +-1,
// an exact multiply.  (The divisions forming alpha and beta run in the tiny
// sb_cg.cu control kernels, so the streaming kernels stay DFMA-free.)
struct DevCoef {
    const double *ptr;
    double scale;
};
__device__ __forceinline__ double coef_value(const DevCoef &c) {
    return c.ptr ? __dmul_rn(c.scale, *c.ptr) : c.scale;
}

// Gated variants used by the device CG (sb_cg.cu): every CTA returns at once
// when *gate == 0, so a converged solve turns later iterations into no-ops.
int cg_axpy(const double *x, double *y, int64_t n, DevCoef a, DevCoef b, const int32_t *gate,
            cudaStream_t st, const char *name);
struct LsaArgs;  // sb_lsa.cuh (multi-GPU combine); nullptr = this rank only
int cg_reduce(int mode, const double *u, const double *v, double *x, double *r, int64_t n, int64_t bs,
              int64_t nb, void *ws, double *result, const int32_t *gate, const double *alpha,
              cudaStream_t st, const char *name, const LsaArgs *lsa = nullptr);
// sb_cg.cu bodies shared by the single- and multi-GPU (sb_lsa_cg_*) entry points
int cg_pap_impl(const double *p, const double *ap, int64_t n, int64_t bs, int64_t nb, void *ws,
                sb_cg_state *st, const LsaArgs *lsa, cudaStream_t s);
int cg_update_impl(int fused, const double *p, const double *ap, double *x, double *r, int64_t n, int64_t bs,
                   int64_t nb, void *ws, sb_cg_state *st, const LsaArgs *lsa, cudaStream_t s);


// ---- cache-policy helpers: HBM streams are touched once -> evict-first.
__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2 *p) { return __ldcs(p); }
__device__ __forceinline__ int4 ld_stream(const int4 *p) { return __ldcs(p); }
__device__ __forceinline__ int ld_stream(const int *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double *p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2 *p, double2 v) { __stcs(p, v); }

// L2 evict_last load for data re-read by later CTAs (BS7 q_global).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_keep(const double *p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ld2_keep(const double *p, uint64_t pol) {
    double2 v;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

// ---- async-copy / mbarrier primitives (sm_90+; used on sm_100a) ----------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile(
        "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(bar)),
        "r"(bytes)
        : "memory");
}
// 8 B shared-memory load at a 32-bit shared address (volatile: stays after
// the mbarrier wait that publishes the data)
__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "SB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra SB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// TMA bulk copy global -> shared (1-D), completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
// TMA bulk copy shared -> global (1-D), tracked by the issuing thread's
// bulk async-groups; the generic-proxy writes to the source must be fenced
// (fence_proxy_async) before the copy is issued.
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// LDGSTS: per-thread async copies tracked by commit/wait groups.
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8_keep(void *dst, const void *src, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace sb
