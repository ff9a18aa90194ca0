// sb_stream.cu -- library plumbing + BS1 copy / BS2 axpy (kernels.py:90-103).
//
// Both are pure HBM streams (16 and 24 B/element).  Design: 128-bit
// (double2) loads/stores, each thread owning U independent double2 per
// stream so ~U*16 B per stream are in flight per thread, one tile of
// 256*U double2 per CTA (no grid-stride tail imbalance), evict-first cache
// policy because every byte is touched once.  A single launch also handles
// the odd head/tail element (block 0, thread 0) so n need not be even.
#include <stdarg.h>
#include <string.h>

#include "sb_common.cuh"

namespace sb {

static thread_local char g_err[512];

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
void clear_error() { g_err[0] = 0; }

int sm_count() {
    static thread_local int dev_cached = -1, sms = kSMs;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return kSMs;
    if (dev != dev_cached) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            sms = v;
        dev_cached = dev;
    }
    return sms;
}

enum ElemOp { OP_COPY = 0, OP_AXPY = 1 };

template <int OP>
__device__ __forceinline__ double elem(double alpha, double x, double beta, double y) {
    if (OP == OP_COPY) return x;
    return add(mul(alpha, x), mul(beta, y));
}

struct ElemDev {
    DevCoef a, b;
    const int32_t *gate;
};

template <int OP, int U, int T, bool DEV = false>
__global__ void __launch_bounds__(T) k_elem_vec(const double2 *x, double2 *y, int64_t n2, double alpha,
                                               double beta, const double *xs, double *ys,
                                               int64_t head_idx, int64_t tail_idx, ElemDev dv = {}) {
    if (DEV) {
        if (*dv.gate == 0) return;
        alpha = coef_value(dv.a);
        beta = coef_value(dv.b);
    }
    const int64_t base = (int64_t)blockIdx.x * (T * U) + threadIdx.x;
    // the odd head / tail element (block 0, thread 0) is loaded with the main
    // stream, not after it: a trailing dependent round trip showed as +0.2 us
    // on every odd n (T0 noise in the size sweeps)
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    double hx = 0.0, hy = 0.0, tx = 0.0, ty = 0.0;
    if (lead) {
        if (head_idx >= 0) {
            hx = xs[head_idx];
            if (OP == OP_AXPY) hy = ys[head_idx];
        }
        if (tail_idx >= 0) {
            tx = xs[tail_idx];
            if (OP == OP_AXPY) ty = ys[tail_idx];
        }
    }
    double2 xv[U], yv[U];
#pragma unroll
    for (int j = 0; j < U; j++) {
        const int64_t i = base + (int64_t)j * T;
        if (i < n2) {
            xv[j] = ld_stream(x + i);
            if (OP == OP_AXPY) yv[j] = ld_stream(y + i);
        }
    }
#pragma unroll
    for (int j = 0; j < U; j++) {
        const int64_t i = base + (int64_t)j * T;
        if (i < n2) {
            double2 o;
            if (OP == OP_COPY) {
                o = xv[j];
            } else {
                o.x = elem<OP>(alpha, xv[j].x, beta, yv[j].x);
                o.y = elem<OP>(alpha, xv[j].y, beta, yv[j].y);
            }
            st_stream(y + i, o);
        }
    }
    if (lead) {
        if (head_idx >= 0) ys[head_idx] = elem<OP>(alpha, hx, beta, hy);
        if (tail_idx >= 0) ys[tail_idx] = elem<OP>(alpha, tx, beta, ty);
    }
}

// Fallback when x and y are not co-aligned to 16 B: scalar grid-stride.
template <int OP, bool DEV = false>
__global__ void __launch_bounds__(256) k_elem_scalar(const double *x, double *y, int64_t n, double alpha,
                                                    double beta, ElemDev dv = {}) {
    if (DEV) {
        if (*dv.gate == 0) return;
        alpha = coef_value(dv.a);
        beta = coef_value(dv.b);
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = elem<OP>(alpha, x[i], beta, y[i]);
}

template <int OP, bool DEV = false>
static int launch_elem(const double *x, double *y, int64_t n, double alpha, double beta,
                       cudaStream_t st, const char *name, ElemDev dv = {}) {
    clear_error();
    if (n < 0 || ((x == nullptr || y == nullptr) && n > 0)) {
        set_error("%s: invalid arguments (n=%lld)", name, (long long)n);
        return SB_E_INVALID;
    }
    if (n == 0) return SB_OK;
    const uintptr_t ax = reinterpret_cast<uintptr_t>(x) & 15u, ay = reinterpret_cast<uintptr_t>(y) & 15u;
    if (ax != ay || (ax & 7u)) {
        const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
        k_elem_scalar<OP, DEV><<<blocks, 256, 0, st>>>(x, y, n, alpha, beta, dv);
        return launch_check(name);
    }
    const int64_t head = ax ? 1 : 0;
    const int64_t n2 = (n - head) / 2;
    const int64_t tail = head + 2 * n2 < n ? head + 2 * n2 : -1;
    constexpr int T = 256, U = 4;
    const int64_t blocks = std::max<int64_t>(1, (n2 + (int64_t)T * U - 1) / ((int64_t)T * U));
    k_elem_vec<OP, U, T, DEV><<<(unsigned)blocks, T, 0, st>>>(
        reinterpret_cast<const double2 *>(x + head), reinterpret_cast<double2 *>(y + head), n2, alpha,
        beta, x, y, head ? 0 : -1, tail, dv);
    return launch_check(name);
}

int cg_axpy(const double *x, double *y, int64_t n, DevCoef a, DevCoef b, const int32_t *gate,
            cudaStream_t st, const char *name) {
    if (!gate) {
        set_error("%s: null gate", name);
        return SB_E_INVALID;
    }
    return launch_elem<OP_AXPY, true>(x, y, n, 0.0, 0.0, st, name, ElemDev{a, b, gate});
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_version(void) { return 100; }

const char *sb_last_error(void) { return sb::g_err; }

int sb_device_info(int device, int *sm, int *major, int *minor, int64_t *l2) {
    clear_error();
    int v;
    if (int rc = cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device), "sm count"))
        return rc;
    if (sm) *sm = v;
    if (major && cuda_check(cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, device), "cc"))
        return SB_E_CUDA;
    if (minor && cuda_check(cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, device), "cc"))
        return SB_E_CUDA;
    if (l2) {
        if (cuda_check(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device), "l2")) return SB_E_CUDA;
        *l2 = v;
    }
    return SB_OK;
}

int sb_bs1_copy(const double *x, double *y, int64_t n, sb_stream_t s) {
    return launch_elem<OP_COPY>(x, y, n, 0.0, 0.0, as_stream(s), "sb_bs1_copy");
}

int sb_bs2_axpy(double alpha, const double *x, double beta, double *y, int64_t n, sb_stream_t s) {
    return launch_elem<OP_AXPY>(x, y, n, alpha, beta, as_stream(s), "sb_bs2_axpy");
}

}  // extern "C"
