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
        set_error("%s: %s", what, cudaGetErrorString(e));
        return SB_E_CUDA;
    }
    return SB_OK;
}

// Launch-error check after <<<>>> (does not synchronise).
inline int launch_check(const char *what) { return cuda_check(cudaGetLastError(), what); }

inline cudaStream_t as_stream(sb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

constexpr int kSMs = 148;  // B200; grids are sized from the device query at runtime

int sm_count();  // cached cudaDevAttrMultiProcessorCount of the current device

// ---- rounded fp64 arithmetic: the reference's numpy temporaries round every
// product and every sum separately; these intrinsics are never contracted.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

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

}  // namespace sb
