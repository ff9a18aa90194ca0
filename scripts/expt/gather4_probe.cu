// TMA tile::gather4 vs LSU gathers (probe, not part of libsb200).
// q viewed as a 2-D tensor [n/2 rows][2 doubles]; entry e needs row col[e] >> 1.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// LSU: one entry per lane, 4 per thread, grid-stride over tiles of 512 entries
__global__ void __launch_bounds__(128) k_ldg(const int32_t *ci, int64_t n, const double *q, double *sink) {
    double acc = 0.0;
    for (int64_t base = (int64_t)blockIdx.x * 512; base < n; base += (int64_t)gridDim.x * 512) {
        int32_t c[4];
#pragma unroll
        for (int j = 0; j < 4; j++) { const int64_t e = base + threadIdx.x + j * 128; c[j] = e < n ? __ldcs(ci + e) : 0; }
        double v[4];
#pragma unroll
        for (int j = 0; j < 4; j++) v[j] = __ldg(q + c[j]);
#pragma unroll
        for (int j = 0; j < 4; j++) acc += v[j];
    }
    if (acc == 1234.5) sink[0] = acc;
}

// TMA: each lane issues one gather4 (4 entries = 4 x 16 B rows) per round;
// a warp moves 128 entries (2 KB) per round, double-buffered.
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap tm, const int32_t *ci, int64_t n,
                                             double *sink) {
    __shared__ __align__(128) double buf[4][2][32 * 16];  // [warp][stage][lane: 128 B slot, 64 B used]
    __shared__ __align__(8) uint64_t bar[4][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int s = 0; s < 2; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    double acc = 0.0;
    const int64_t nw = (int64_t)gridDim.x * 4;
    uint32_t ph[2] = {0, 0};
    auto issue = [&](int64_t r, int s) {
        const int64_t base = (r * nw + blockIdx.x * 4 + warp) * 128;
        if (base >= n) return false;
        int32_t rows[4];
#pragma unroll
        for (int j = 0; j < 4; j++) { const int64_t e = base + lane * 4 + j; rows[j] = e < n ? (__ldcs(ci + e) >> 1) : 0; }
        if (lane == 0)
            asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
                             smem_u32(&bar[warp][s])), "r"(128 * 16) : "memory");
        __syncwarp();
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(smem_u32(&buf[warp][s][lane * 16])), "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]),
              "r"(smem_u32(&bar[warp][s])) : "memory");
        return true;
    };
    bool live[2];
    live[0] = issue(0, 0);
    live[1] = issue(1, 1);
    for (int64_t r = 0;; r++) {
        const int s = (int)(r & 1);
        if (!live[s]) break;
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                     ::"r"(smem_u32(&bar[warp][s])), "r"(ph[s]) : "memory");
        ph[s] ^= 1;
#pragma unroll
        for (int j = 0; j < 8; j++) acc += buf[warp][s][lane * 16 + j];
        __syncwarp();
        live[s] = issue(r + 2, s);
    }
    if (acc == 1234.5) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int probe(int mode, const int32_t *ci, int64_t n, const double *q, int64_t nq, double *sink, int grid,
                     void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (mode == 0) {
        k_ldg<<<grid, 128, 0, st>>>(ci, n, q, sink);
        return (int)cudaGetLastError();
    }
    static CUtensorMap tm;
    static const double *tq = nullptr;
    if (tq != q) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn) return -2;
        cuuint64_t gdim[2] = {2, (cuuint64_t)(nq / 2)};
        cuuint64_t gstr[1] = {16};
        cuuint32_t box[2] = {2, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)q, gdim, gstr, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return -3 - (int)r;
        tq = q;
    }
    k_tma<<<grid, 128, 0, st>>>(tm, ci, n, sink);
    return (int)cudaGetLastError();
}
