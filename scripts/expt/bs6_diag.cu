// BS6 bottleneck diagnosis (not part of libsb200): the product kernel with
// (QSEQ) the q gather replaced by a sequential read of the same bytes and/or
// (SUMS=false) the serial row sums replaced by one shared-memory read, plus a
// pure streaming kernel moving BS6's byte mix (the ceiling for this traffic).
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
__device__ __forceinline__ int ld_stream(const int *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double *p, double v) { __stcs(p, v); }
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

// Shared-memory slot of super-block entry k.  With long rows (p = 1: 8
// entries) the one-thread-per-row sums read qs[8l + j] across lanes l -- a
// 16-way bank conflict; XOR-ing the low 4 bits of the double index with bits
// 4..7 makes those reads 2 wavefronts (the minimum for 32 x 8 B).  Rows of
// length 1-2 (p >= 3) are already conflict-light, so SWZ is chosen per
// operator from the mean row length.
template <bool SWZ>
__device__ __forceinline__ int qslot(int k) {
    return SWZ ? (k ^ ((k >> 4) & 15)) : k;
}

template <int T, int CAP, bool SWZ, int QSEQ, bool SUMS>
__global__ void __launch_bounds__(T, 12) k_diag(const int32_t *__restrict__ plan, int64_t nsb,
                                                            const int32_t *__restrict__ rs,
                                                            const int32_t *__restrict__ ci,
                                                            const double *__restrict__ q,
                                                            double *__restrict__ out,
                                                            const double *__restrict__ carry, int64_t ncarry, int zero) {
    constexpr int M = CAP / (2 * T);          // entry pairs per thread
    constexpr int R = (CAP + 1 + T - 1) / T;  // row starts per thread (rows <= CAP)
    extern __shared__ __align__(16) unsigned char bs6_smem[];
    double(*qs)[CAP] = reinterpret_cast<double(*)[CAP]>(bs6_smem);
    int32_t(*rss)[CAP + 4] = reinterpret_cast<int32_t(*)[CAP + 4]>(bs6_smem + 2 * CAP * sizeof(double));

    const int64_t g = gridDim.x;
    int64_t sbi = blockIdx.x;
    SbMeta mc = load_meta(plan, sbi, nsb);      // current super-block
    SbMeta mn = load_meta(plan, sbi + g, nsb);  // next
    int2 cols[M];  // each thread owns consecutive entries (2k, 2k+1)
#pragma unroll
    for (int m = 0; m < M; m++) {
        const int k = 2 * (threadIdx.x + m * T), ne = mc.e1 - mc.e0;
        if (k < ne) cols[m].x = ld_stream(ci + mc.e0 + k);
        if (k + 1 < ne) cols[m].y = ld_stream(ci + mc.e0 + k + 1);
    }
    int buf = 0;
    for (; sbi < nsb; sbi += g) {
        const int ne = mc.e1 - mc.e0, nrows = mc.r1 - mc.r0;
        // A: value gathers of this super-block -- one 16 B load when the pair's
        //    columns are consecutive (an element edge), else two 8 B loads
        double2 v[M];
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = 2 * (threadIdx.x + m * T);
            if (k + 1 < ne) {
                if (QSEQ) { v[m] = __ldg(reinterpret_cast<const double2 *>(q + mc.e0 + k - ((mc.e0+k)&1) + (cols[m].x & zero) + (cols[m].y & zero))); } else if (cols[m].y == cols[m].x + 1 && aligned16(q + cols[m].x)) {
                    v[m] = __ldg(reinterpret_cast<const double2 *>(q + cols[m].x));
                } else {
                    v[m].x = __ldg(q + cols[m].x);
                    v[m].y = __ldg(q + cols[m].y);
                }
            } else if (k < ne) {
                v[m].x = __ldg(q + cols[m].x);
            }
        }
        // B: row starts of this super-block
        int32_t rv[R];
#pragma unroll
        for (int j = 0; j < R; j++) {
            const int k = threadIdx.x + j * T;
            if (k <= nrows) rv[j] = ld_stream(rs + mc.r0 + k);
        }
        // C: indices of the next super-block; D: plan entry of the one after
        const int nne = mn.e1 - mn.e0;
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = 2 * (threadIdx.x + m * T);
            if (k < nne) cols[m].x = ld_stream(ci + mn.e0 + k);
            if (k + 1 < nne) cols[m].y = ld_stream(ci + mn.e0 + k + 1);
        }
        const SbMeta mnn = load_meta(plan, sbi + 2 * g, nsb);
        // E: publish A/B to shared memory
#pragma unroll
        for (int m = 0; m < M; m++) {
            const int k = 2 * (threadIdx.x + m * T);
            if (SWZ) {
                if (k < ne) qs[buf][qslot<SWZ>(k)] = v[m].x;
                if (k + 1 < ne) qs[buf][qslot<SWZ>(k + 1)] = v[m].y;
            } else if (k + 1 < ne) {
                *reinterpret_cast<double2 *>(&qs[buf][k]) = v[m];
            } else if (k < ne) {
                qs[buf][k] = v[m].x;
            }
        }
#pragma unroll
        for (int j = 0; j < R; j++) {
            const int k = threadIdx.x + j * T;
            if (k <= nrows) rss[buf][k] = rv[j];
        }
        __syncthreads();
        // G: one thread per row, ascending column order
        for (int k = threadIdx.x; k < nrows; k += T) {
            const int a = rss[buf][k] - mc.e0, b = rss[buf][k + 1] - mc.e0;
            const int64_t r = (int64_t)mc.r0 + k;
            double acc = r < ncarry ? carry[r] : 0.0;
            if (SUMS) { for (int c = a; c < b; c++) acc = add(acc, qs[buf][qslot<SWZ>(c)]); } else acc = qs[buf][qslot<SWZ>(a)];
            st_stream(out + r, acc);
        }
        buf ^= 1;  // the barrier of the next iteration separates reuse of this buffer
        mc = mn;
        mn = mnn;
    }
}


// ceiling: read q (NL f64), ci (NL i32), rs (NG i32) sequentially, write out (NG f64)
__global__ void __launch_bounds__(256) k_ceiling(const double2 *q, const int2 *ci, const int2 *rs, double2 *out,
                                                 int64_t nl2, int64_t ng2) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl2; i += (int64_t)gridDim.x * blockDim.x) {
        double2 a = __ldcs(q + i);
        int2 c = __ldcs(ci + i);
        double s = a.x + a.y + c.x + c.y;
        if (i < ng2) {
            int2 r = __ldcs(rs + i);
            __stcs(out + i, make_double2(s, (double)r.x + r.y));
        } else if (s == 12345.678) {
            out[0].x = s;
        }
    }
}

template <int QSEQ, bool SUMS, bool SWZ>
static void run(const int32_t *plan, int64_t nsb, const int32_t *rs, const int32_t *ci, const double *q,
                double *out, cudaStream_t st) {
    constexpr int T = 128, CAP = 512;
    const size_t smem = 2 * CAP * sizeof(double) + 2 * (CAP + 4) * sizeof(int32_t);
    auto kern = k_diag<T, CAP, SWZ, QSEQ, SUMS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    const int64_t grid = std::min<int64_t>(nsb, 148LL * per_sm);
    kern<<<(unsigned)grid, T, smem, st>>>(plan, nsb, rs, ci, q, out, nullptr, 0, 0);
}

extern "C" int diag_bs6(int variant, const int32_t *plan, int64_t nsb, const int32_t *rs, const int32_t *ci,
                        const double *q, double *out, int64_t nl, int64_t ng, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    switch (variant) {
        case 0: run<0, true, false>(plan, nsb, rs, ci, q, out, st); break;
        case 1: run<1, true, false>(plan, nsb, rs, ci, q, out, st); break;
        case 2: run<0, false, false>(plan, nsb, rs, ci, q, out, st); break;
        case 3: run<1, false, false>(plan, nsb, rs, ci, q, out, st); break;
        case 4: k_ceiling<<<148 * 16, 256, 0, st>>>((const double2 *)q, (const int2 *)ci, (const int2 *)rs,
                                                    (double2 *)out, nl / 2, ng / 2); break;
        default: return -1;
    }
    return (int)cudaGetLastError();
}
