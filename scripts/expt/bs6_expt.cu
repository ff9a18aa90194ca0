// Experimental BS6 variants for A/B timing on the box (not part of libsb200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o expt.so bs6_expt.cu
// Variant flags: SUMS (do the row sums), CONTIG (contiguous super-block ranges
// per CTA instead of round-robin).
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

struct SbMeta {
    int32_t r0, e0, r1, e1;
};

__device__ __forceinline__ SbMeta load_meta(const int32_t *plan, int64_t i, int64_t nsb) {
    SbMeta m{0, 0, 0, 0};
    if (i < nsb) {
        const int2 lo = __ldg(reinterpret_cast<const int2 *>(plan + 2 * i));
        const int2 hi = __ldg(reinterpret_cast<const int2 *>(plan + 2 * i + 2));
        m = SbMeta{lo.x, lo.y, hi.x, hi.y};
    }
    return m;
}

template <int T, int CAP, bool SUMS, bool CONTIG, int MINB>
__global__ void __launch_bounds__(T, MINB) k_pipe(const int32_t *__restrict__ plan, int64_t nsb,
                                                  const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                                                  const double *__restrict__ q, double *__restrict__ out) {
    constexpr int M = CAP / T;
    constexpr int R = (CAP + 1 + T - 1) / T;
    extern __shared__ __align__(16) unsigned char smem[];
    double(*qs)[CAP] = reinterpret_cast<double(*)[CAP]>(smem);
    int32_t(*rss)[CAP + 4] = reinterpret_cast<int32_t(*)[CAP + 4]>(smem + 2 * CAP * sizeof(double));
    int64_t g, sbi, send;
    if (CONTIG) {
        const int64_t per = (nsb + gridDim.x - 1) / gridDim.x;
        sbi = blockIdx.x * per;
        send = sbi + per < nsb ? sbi + per : nsb;
        g = 1;
    } else {
        sbi = blockIdx.x;
        send = nsb;
        g = gridDim.x;
    }
    SbMeta mc = load_meta(plan, sbi, send);
    SbMeta mn = load_meta(plan, sbi + g, send);
    int32_t cols[M];
#pragma unroll
    for (int m = 0; m < M; m++) {
        const int k = threadIdx.x + m * T;
        if (k < mc.e1 - mc.e0) cols[m] = __ldcs(ci + mc.e0 + k);
    }
    int buf = 0;
    for (; sbi < send; sbi += g) {
        const int ne = mc.e1 - mc.e0, nrows = mc.r1 - mc.r0;
        double v[M];
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = threadIdx.x + m * T;
            if (k < ne) v[m] = __ldg(q + cols[m]);
        }
        int32_t rv[R];
#pragma unroll
        for (int j = 0; j < R; j++) {
            const int k = threadIdx.x + j * T;
            if (k <= nrows) rv[j] = __ldcs(rs + mc.r0 + k);
        }
        const int nne = mn.e1 - mn.e0;
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = threadIdx.x + m * T;
            if (k < nne) cols[m] = __ldcs(ci + mn.e0 + k);
        }
        const SbMeta mnn = load_meta(plan, sbi + 2 * g, send);
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = threadIdx.x + m * T;
            if (k < ne) qs[buf][k] = v[m];
        }
#pragma unroll
        for (int j = 0; j < R; j++) {
            const int k = threadIdx.x + j * T;
            if (k <= nrows) rss[buf][k] = rv[j];
        }
        __syncthreads();
        for (int k = threadIdx.x; k < nrows; k += T) {
            double acc = 0.0;
            if (SUMS) {
                const int a = rss[buf][k] - mc.e0, b = rss[buf][k + 1] - mc.e0;
                for (int c = a; c < b; c++) acc = add(acc, qs[buf][c]);
            } else {
                acc = qs[buf][k];
            }
            __stcs(out + mc.r0 + k, acc);
        }
        buf ^= 1;
        mc = mn;
        mn = mnn;
    }
}

// pairs of consecutive entries per thread; 16 B gathers when the two columns are consecutive
template <int T, int CAP, int MINB>
__global__ void __launch_bounds__(T, MINB) k_pipe2(const int32_t *__restrict__ plan, int64_t nsb,
                                                   const int32_t *__restrict__ rs, const int32_t *__restrict__ ci,
                                                   const double *__restrict__ q, double *__restrict__ out) {
    constexpr int M = CAP / (2 * T);  // pairs per thread
    constexpr int R = (CAP + 1 + T - 1) / T;
    extern __shared__ __align__(16) unsigned char smem[];
    double(*qs)[CAP] = reinterpret_cast<double(*)[CAP]>(smem);
    int32_t(*rss)[CAP + 4] = reinterpret_cast<int32_t(*)[CAP + 4]>(smem + 2 * CAP * sizeof(double));
    const int64_t g = gridDim.x;
    int64_t sbi = blockIdx.x;
    SbMeta mc = load_meta(plan, sbi, nsb), mn = load_meta(plan, sbi + g, nsb);
    int2 cols[M];
#pragma unroll
    for (int m = 0; m < M; m++) {
        const int k = 2 * (threadIdx.x + m * T);
        const int ne = mc.e1 - mc.e0;
        if (k < ne) cols[m].x = __ldcs(ci + mc.e0 + k);
        if (k + 1 < ne) cols[m].y = __ldcs(ci + mc.e0 + k + 1);
    }
    int buf = 0;
    for (; sbi < nsb; sbi += g) {
        const int ne = mc.e1 - mc.e0, nrows = mc.r1 - mc.r0;
        double2 v[M];
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = 2 * (threadIdx.x + m * T);
            if (k + 1 < ne) {
                if (cols[m].y == cols[m].x + 1 && (cols[m].x & 1) == 0) {
                    v[m] = __ldg(reinterpret_cast<const double2 *>(q + cols[m].x));
                } else {
                    v[m].x = __ldg(q + cols[m].x);
                    v[m].y = __ldg(q + cols[m].y);
                }
            } else if (k < ne) {
                v[m].x = __ldg(q + cols[m].x);
            }
        }
        int32_t rv[R];
#pragma unroll
        for (int j = 0; j < R; j++) {
            const int k = threadIdx.x + j * T;
            if (k <= nrows) rv[j] = __ldcs(rs + mc.r0 + k);
        }
        const int nne = mn.e1 - mn.e0;
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = 2 * (threadIdx.x + m * T);
            if (k < nne) cols[m].x = __ldcs(ci + mn.e0 + k);
            if (k + 1 < nne) cols[m].y = __ldcs(ci + mn.e0 + k + 1);
        }
        const SbMeta mnn = load_meta(plan, sbi + 2 * g, nsb);
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = 2 * (threadIdx.x + m * T);
            if (k + 1 < ne) *reinterpret_cast<double2 *>(&qs[buf][k]) = v[m];
            else if (k < ne) qs[buf][k] = v[m].x;
        }
#pragma unroll
        for (int j = 0; j < R; j++) {
            const int k = threadIdx.x + j * T;
            if (k <= nrows) rss[buf][k] = rv[j];
        }
        __syncthreads();
        for (int k = threadIdx.x; k < nrows; k += T) {
            double acc = 0.0;
            const int a = rss[buf][k] - mc.e0, b = rss[buf][k + 1] - mc.e0;
            for (int c = a; c < b; c++) acc = add(acc, qs[buf][c]);
            __stcs(out + mc.r0 + k, acc);
        }
        buf ^= 1;
        mc = mn;
        mn = mnn;
    }
}

template <int CAP, int MINB, int T>
static int run2(const int32_t *plan, int64_t nsb, const int32_t *rs, const int32_t *ci, const double *q, double *out,
                cudaStream_t st) {
    const size_t smem = 2 * CAP * sizeof(double) + 2 * (CAP + 4) * sizeof(int32_t);
    cudaFuncSetAttribute(k_pipe2<T, CAP, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pipe2<T, CAP, MINB>, T, smem);
    int64_t grid = 148LL * per_sm;
    if (grid > nsb) grid = nsb;
    k_pipe2<T, CAP, MINB><<<(unsigned)grid, T, smem, st>>>(plan, nsb, rs, ci, q, out);
    return per_sm;
}

template <int CAP, bool SUMS, bool CONTIG, int MINB, int T = 256>
static int run(const int32_t *plan, int64_t nsb, const int32_t *rs, const int32_t *ci, const double *q, double *out,
               int ctas_per_sm, cudaStream_t st) {
    const size_t smem = 2 * CAP * sizeof(double) + 2 * (CAP + 4) * sizeof(int32_t);
    cudaFuncSetAttribute(k_pipe<T, CAP, SUMS, CONTIG, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pipe<T, CAP, SUMS, CONTIG, MINB>, T, smem);
    if (ctas_per_sm > 0 && ctas_per_sm < per_sm) per_sm = ctas_per_sm;
    int64_t grid = 148LL * per_sm;
    (void)0;
    if (grid > nsb) grid = nsb;
    k_pipe<T, CAP, SUMS, CONTIG, MINB><<<(unsigned)grid, T, smem, st>>>(plan, nsb, rs, ci, q, out);
    return per_sm;
}

extern "C" int expt_bs6(int variant, const int32_t *plan, int64_t nsb, const int32_t *rs, const int32_t *ci,
                        const double *q, double *out, int ctas_per_sm, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    switch (variant) {
        case 0: return run<2048, true, false, 3>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 1: return run<2048, false, false, 3>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 2: return run<2048, true, true, 3>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 3: return run<1024, true, false, 4>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 4: return run<1024, true, true, 4>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 5: return run<512, true, false, 6>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 6: return run<512, true, false, 8>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 7: return run<512, true, false, 12, 128>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 8: return run<256, true, false, 16, 128>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 9: return run<1024, true, false, 4, 512>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 10: return run<1024, true, false, 6, 256>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 11: return run<512, false, false, 8>(plan, nsb, rs, ci, q, out, ctas_per_sm, st);
        case 12: return run2<512, 12, 128>(plan, nsb, rs, ci, q, out, st);
        case 13: return run2<512, 16, 128>(plan, nsb, rs, ci, q, out, st);
        case 14: return run2<1024, 8, 256>(plan, nsb, rs, ci, q, out, st);
        default: return -1;
    }
}
