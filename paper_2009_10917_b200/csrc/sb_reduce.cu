// sb_reduce.cu -- BS3 norm, BS4 dot, BS5 fused CG update (kernels.py:19-132).
//
// The reference fixes the reduction *schedule* (kernels.py:38-87, the paper's
// Listing 3): S = block_size*n_blocks lattice slots; slot s accumulates
// u[s + c*S]*v[s + c*S] for c = 0,1,.. in order from +0.0 (rounded product,
// rounded add); a power-of-two tree folds each block's block_size slots to one
// partial; one block of block_size slots folds the n_blocks partials
// (sequential per slot, then the same tree).  We reproduce it bit for bit:
//
//   * CTA b <-> lattice block b, thread t owns slots t + j*T (j < SPT,
//     block_size = T*SPT), so for every step c a warp reads 32 consecutive
//     doubles (coalesced) and the per-slot order is the reference's.
//   * Memory-level parallelism comes from unrolling the chain by U steps:
//     all U*streams loads are issued before the U in-order adds.
//   * Tree: shared memory for levels k >= 32, warp shuffles for 16..1 --
//     level k adds slot s+k into slot s exactly as `rows[:k] += rows[k:2k]`.
//   * Single launch: every CTA but 0 publishes its block value(s) as flagged
//     8-byte words (no fence, no atomic); CTA 0 runs the second stage from
//     them as they arrive and re-zeroes the slots (second_stage below).
//   * BS5 updates x and r and accumulates r_new^2 in the same pass (48 B/el,
//     the reference's CPU code re-reads r), on the BS3 lattice, so
//     bs5 == bs3_norm2(r_new) bitwise (test_kernels.py:194-199).
#include <stdlib.h>

#include <algorithm>

#include "sb_common.cuh"
#include "sb_lsa.cuh"

namespace sb {

// Ring shapes (bytes of stages per CTA, chain steps per stage); overridable at
// build time for the A/B sweeps in scripts/expt/run_lattice.py.
#ifndef SB_SPS_NORM
#define SB_SPS_NORM 8
#define SB_SPS_DOT 4
#define SB_SPS_FUSED 2
#define SB_RING_NORM 32768
#define SB_RING_DOT 32768
#define SB_RING_FUSED 32768
#endif
#ifndef SB_BPC
#define SB_BPC 1
#endif

constexpr int kBpc = SB_BPC;  // lattice blocks per CTA for block_size 256 (A/B)
constexpr int kSpsNorm = SB_SPS_NORM, kSpsDot = SB_SPS_DOT, kSpsFused = SB_SPS_FUSED;
constexpr int kRingNorm = SB_RING_NORM, kRingDot = SB_RING_DOT, kRingFused = SB_RING_FUSED;
#ifndef SB_RING_FUSED_BPC4
#define SB_RING_FUSED_BPC4 131072
#endif
constexpr int kRingFusedBpc4 = SB_RING_FUSED_BPC4;  // 4 stages of 4 arrays x 8 KB


enum RMode { R_NORM = 0, R_DOT = 1, R_FUSED = 2 };

struct RArgs {
    const double *u;  // NORM/DOT: x ; FUSED: p
    const double *v;  // DOT: y      ; FUSED: ap
    double *x;        // FUSED
    double *r;        // FUSED
    double alpha;
    int64_t n;
    int64_t S;   // block_size * n_blocks
    int64_t bs;  // block_size
    int64_t nb;  // n_blocks
    double *partials;
    unsigned long long *ll;  // flagged partial slots, 16 B per lattice block
    double *result;
    double *lattice;  // generic path only
    // device CG: *gate == 0 -> every CTA returns; alpha read from *alpha_ptr
    const int32_t *gate;
    const double *alpha_ptr;
    // multi-GPU fused combine (sb_lsa.cuh): the last CTA publishes the rank's
    // scalar to every NVLink peer and sums the ranks' scalars in rank order
    LsaArgs lsa;
};

// Thread 0 of the last CTA: write the block-reduced scalar.
__device__ __forceinline__ void write_result(const RArgs &A, double v) {
    if (A.lsa.enabled)
        *A.result = lsa_combine(A.lsa, v);
    else
        *A.result = v;
}

// Gate check + device alpha at kernel entry (a no-op for plain calls).
__device__ __forceinline__ bool resolve(RArgs &A) {
    if (A.gate && *A.gate == 0) return false;
    if (A.alpha_ptr) A.alpha = *A.alpha_ptr;
    return true;
}

// Workspace layout: [256 B header (sb_dot_compensated's ticket)][partials:
// nb doubles (generic path)][flagged partial
// slots: nb x 16 B][generic path: S + bs doubles].  Zero between calls.
static size_t ll_offset(int64_t nb) { return (256 + sizeof(double) * (size_t)nb + 15) & ~(size_t)15; }  // 16 B aligned
static size_t ws_bytes(int64_t bs, int64_t nb) {
    size_t b = ll_offset(nb) + 16 * (size_t)nb;
    if (bs > 1024) b += sizeof(double) * ((size_t)bs * (size_t)nb + (size_t)bs);
    return (b + 255) & ~(size_t)255;
}

// One chain step for slot value(s) at element i.
template <int MODE>
struct Step;

template <>
struct Step<R_NORM> {
    double a;
    __device__ __forceinline__ void load(const RArgs &A, int64_t i) { a = ld_stream(A.u + i); }
    __device__ __forceinline__ double term(const RArgs &) const { return mul(a, a); }
    __device__ __forceinline__ void pin() { asm volatile("" : "+d"(a)); }
};
template <>
struct Step<R_DOT> {
    double a, b;
    __device__ __forceinline__ void load(const RArgs &A, int64_t i) {
        a = ld_stream(A.u + i);
        b = ld_stream(A.v + i);
    }
    __device__ __forceinline__ double term(const RArgs &) const { return mul(a, b); }
    __device__ __forceinline__ void pin() { asm volatile("" : "+d"(a), "+d"(b)); }
};
template <>
struct Step<R_FUSED> {
    double p, ap, x, r;
    __device__ __forceinline__ void load(const RArgs &A, int64_t i) {
        p = ld_stream(A.u + i);
        ap = ld_stream(A.v + i);
        x = ld_stream(A.x + i);
        r = ld_stream(A.r + i);
    }
    __device__ __forceinline__ void pin() { asm volatile("" : "+d"(p), "+d"(ap), "+d"(x), "+d"(r)); }
    // x += alpha*p ; r -= alpha*ap (kernels.py:127-131); returns r_new^2
    __device__ __forceinline__ double update_store(const RArgs &A, int64_t i) {
        const double xn = add(x, mul(A.alpha, p));
        const double rn = sub(r, mul(A.alpha, ap));
        st_stream(A.x + i, xn);
        st_stream(A.r + i, rn);
        return mul(rn, rn);
    }
};

template <int MODE>
__device__ __forceinline__ double step_term(Step<MODE> &s, const RArgs &A, int64_t i) {
    if constexpr (MODE == R_FUSED)
        return s.update_store(A, i);
    else
        return s.term(A);
}

// Fold `bs` slots held in shared memory (sm[0..bs)) with the reference tree;
// returns the block value in thread 0.  T threads participate.
template <int T>
__device__ __forceinline__ double tree_fold(double *sm, int bs) {
    for (int k = bs / 2; k >= 32; k >>= 1) {
        for (int s = threadIdx.x; s < k; s += T) sm[s] = add(sm[s], sm[s + k]);
        __syncthreads();
    }
    double v = 0.0;
    if (threadIdx.x < 32) {
        const int w = bs < 32 ? bs : 32;
        const unsigned mask = T >= 32 ? 0xffffffffu : ((1u << T) - 1u);
        if ((int)threadIdx.x < w) v = sm[threadIdx.x];
        for (int off = w / 2; off >= 1; off >>= 1) v = add(v, __shfl_down_sync(mask, v, off));
    }
    return v;
}

// Cross-CTA combine of k_lattice without a ticket: every CTA but 0 publishes
// its block value as two 8-byte words {flag = 1, 32-bit half} (each word is
// single-copy atomic, so a reader that sees the flag sees its half -- no
// fence, no atomic), and CTA 0 runs the second stage straight from those
// slots, spinning on each until it is flagged, then zeroes it for the next
// call.  One L2 round trip less than release-ticket + re-read; no deadlock
// risk: only CTA 0 waits, and every other CTA runs to completion without
// waiting on anything.
__device__ __forceinline__ void ll_put(unsigned long long *slot, double v) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const unsigned long long hi = (1ull << 32) | (bits >> 32), lo = (1ull << 32) | (bits & 0xffffffffull);
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(hi), "l"(lo) : "memory");
}
// Poll bound of ll_take (0 = wait forever, the default): a debug aid set from
// SB200_POLL_LIMIT (polls; ~256 ns each after the first 4096).  A slow but
// correct reduction -- CTAs starved by concurrent kernels, MPS partitions, a
// sanitizer -- must not turn into a sticky launch failure.
__device__ unsigned long long g_sb_poll_limit = 0;

__device__ __forceinline__ double ll_take(unsigned long long *slot) {
    unsigned long long hi, lo;
    const unsigned long long limit = g_sb_poll_limit;
    for (unsigned long long polls = 0;; polls++) {
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(hi), "=l"(lo) : "l"(slot) : "memory");
        if ((hi >> 32) == 1ull && (lo >> 32) == 1ull) break;
        if (polls >= 4096) __nanosleep(256);
        if (limit && polls == limit) __trap();
    }
    asm volatile("st.global.v2.u64 [%0], {%1, %1};" ::"l"(slot), "l"(0ull) : "memory");
    return __longlong_as_double((long long)(((hi & 0xffffffffull) << 32) | (lo & 0xffffffffull)));
}

template <int T>
__device__ __forceinline__ void second_stage(const RArgs &A, double *sm, int bs, int spt, double v) {
    if (blockIdx.x != 0) {
        if (threadIdx.x == 0) ll_put(A.ll + 2 * blockIdx.x, v);
        return;
    }
    // _final_reduce (kernels.py:72-81): s[t] = 0.0 + partials[t] + partials[t+bs] + ...
    // over the launched blocks (see launch_reduce: blocks past n hold +0.0,
    // and acc + 0.0 == acc for an acc that started at +0.0); partial 0 is
    // this CTA's own value, held by thread 0 (the owner of slot 0)
    for (int j = 0; j < spt; j++) {
        const int t = threadIdx.x + j * T;
        double acc = 0.0;
        for (int64_t c = t; c < (int64_t)gridDim.x; c += bs)
            acc = add(acc, c == 0 ? v : ll_take(A.ll + 2 * c));
        sm[t] = acc;
    }
    __syncthreads();
    const double res = tree_fold<T>(sm, bs);
    if (threadIdx.x == 0) write_result(A, res);
}

// The last, partial batch of a chain (fewer than U steps left): all of its
// loads first, then the in-order adds (and BS5's stores), so a ragged chain
// costs one memory latency instead of one per remaining step.  The batch
// ends with a branch at the first step past n rather than predicating every
// load: U*SPT live predicates would not fit the 7 predicate registers (the
// compiler then splits the batch), and clamped re-loads of a valid element
// hot-spot one L2 slice when every thread's chain is short (n < S).
template <int T, int SPT, int MODE, int U>
__device__ __forceinline__ void ragged_batch(const RArgs &A, int64_t c0, double (&acc)[SPT]) {
    const int64_t S = A.S, n = A.n;
    Step<MODE> st[U][SPT];
#pragma unroll
    for (int k = 0; k < U; k++) {
        const int64_t ik = c0 + (int64_t)k * S;
        if (ik >= n) break;
#pragma unroll
        for (int j = 0; j < SPT; j++)
            if (ik + (int64_t)j * T < n) st[k][j].load(A, ik + (int64_t)j * T);
    }
    // keep the compiler from hoisting step 0's arithmetic between the loads
    // of the later steps (it knows step 0 exists; BS5 otherwise loses a latency)
#pragma unroll
    for (int k = 0; k < U; k++)
#pragma unroll
        for (int j = 0; j < SPT; j++) st[k][j].pin();
#pragma unroll
    for (int k = 0; k < U; k++) {
        const int64_t ik = c0 + (int64_t)k * S;
        if (ik >= n) break;
#pragma unroll
        for (int j = 0; j < SPT; j++) {
            const int64_t i = ik + (int64_t)j * T;
            if (i < n) acc[j] = add(acc[j], step_term<MODE>(st[k][j], A, i));
        }
    }
}

template <int T, int SPT, int MODE, int U>
__global__ void __launch_bounds__(T, (1024 / T) < 32 ? (1024 / T) : 32) k_lattice(RArgs Ain) {
    RArgs A = Ain;
    if (!resolve(A)) return;
    __shared__ double sm[T * SPT];
    const int bs = T * SPT;
    const int64_t slot0 = (int64_t)blockIdx.x * bs + threadIdx.x;
    double acc[SPT];
#pragma unroll
    for (int j = 0; j < SPT; j++) acc[j] = 0.0;

    const int64_t S = A.S, n = A.n;
    int64_t c0 = slot0;
    // full batches: every (k, j) element of the batch exists
    const int64_t last_off = (int64_t)(U - 1) * S + (int64_t)(SPT - 1) * T;
    for (; c0 + last_off < n; c0 += (int64_t)U * S) {
        Step<MODE> st[U][SPT];
#pragma unroll
        for (int k = 0; k < U; k++)
#pragma unroll
            for (int j = 0; j < SPT; j++) st[k][j].load(A, c0 + (int64_t)k * S + (int64_t)j * T);
#pragma unroll
        for (int k = 0; k < U; k++)
#pragma unroll
            for (int j = 0; j < SPT; j++)
                acc[j] = add(acc[j], step_term<MODE>(st[k][j], A, c0 + (int64_t)k * S + (int64_t)j * T));
    }
    // fewer than U steps are left (c0 + U*S > n, as S > (SPT-1)*T): one more
    // batch, in its own (non-inlined) function so it does not perturb the
    // register allocation and load-then-add schedule of the loop above
    if (c0 < n) ragged_batch<T, SPT, MODE, U>(A, c0, acc);
#pragma unroll
    for (int j = 0; j < SPT; j++) sm[threadIdx.x + j * T] = acc[j];
    __syncthreads();
    const double v = tree_fold<T>(sm, bs);
    __syncthreads();
    second_stage<T>(A, sm, bs, SPT, v);
}

// ---- TMA-ring lattice kernel ---------------------------------------------
// Same lattice, same per-slot order; the memory-level parallelism comes from a
// ring of ST shared-memory stages filled by cp.async.bulk (TMA) instead of
// registers.  For step c, CTA b's slots need the contiguous chunk
// [c*S + b*bs, +bs) of every input array -- one bulk copy per array per
// stage, issued by a dedicated producer warp.  The T/32 consumer warps read
// their slots from shared memory, fold them into their chains in c order and
// (BS5) stream x', r' back with evict-first stores; each consumer warp
// releases the stage through an `empty` mbarrier.  The last (partial) chunk
// of a CTA, if any, is read straight from global memory, still in chain order.
template <int MODE>
struct NArr {
    static constexpr int v = MODE == R_NORM ? 1 : (MODE == R_DOT ? 2 : 4);
};

template <int T, int SPT, int MODE, int ST, int SPS, int BPC = 1>
__global__ void __launch_bounds__(T + 32) k_lattice_tma(RArgs Ain) {
    RArgs A = Ain;
    if (!resolve(A)) return;
    // A stage holds SPS consecutive chain steps (chunks) of every array, so
    // the per-byte cost of the full/empty handshakes drops by SPS.
    constexpr int BS = T * SPT;
    constexpr int NA = NArr<MODE>::v;
    constexpr int NCW = T / 32;  // consumer warps
    extern __shared__ __align__(128) unsigned char lat_smem[];  // ST stages, dynamic
    double(*buf)[SPS][NA][BS] = reinterpret_cast<double(*)[SPS][NA][BS]>(lat_smem);
    __shared__ __align__(8) uint64_t full[ST], empty[ST];
    __shared__ double sm[BS];

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t S = A.S, n = A.n;
    const int64_t base0 = (int64_t)blockIdx.x * BS;
    const int64_t nfull = n >= base0 + BS ? (n - base0 - BS) / S + 1 : 0;
    const int64_t nstage = nfull / SPS;

    if (tid == 0) {
        for (int s = 0; s < ST; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    double acc[SPT];
#pragma unroll
    for (int j = 0; j < SPT; j++) acc[j] = 0.0;

    if (warp == NCW) {
        // producer warp: one elected lane issues the bulk copies
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const double *src[4] = {A.u, A.v, A.x, A.r};
            int s = 0;
            uint32_t ph = 0;  // parity of the current pass over the ring
            for (int64_t c = 0; c < nstage; c++) {
                if (c >= ST) mbar_wait(&empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&full[s], (uint32_t)(SPS * NA * BS * sizeof(double)));
#pragma unroll
                for (int u = 0; u < SPS; u++) {
                    const int64_t off = (c * SPS + u) * S + base0;
#pragma unroll
                    for (int a = 0; a < NA; a++)
                        bulk_g2s(&buf[s][u][a][0], src[a] + off, (uint32_t)(BS * sizeof(double)), &full[s], pol);
                }
                if (++s == ST) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
    } else {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t c = 0; c < nstage; c++) {
            mbar_wait(&full[s], ph);
#pragma unroll
            for (int u = 0; u < SPS; u++) {
                const int64_t off = (c * SPS + u) * S + base0;
#pragma unroll
                for (int j = 0; j < SPT; j++) {
                    const int k = tid + j * T;
                    if constexpr (MODE == R_NORM) {
                        const double a = buf[s][u][0][k];
                        acc[j] = add(acc[j], mul(a, a));
                    } else if constexpr (MODE == R_DOT) {
                        acc[j] = add(acc[j], mul(buf[s][u][0][k], buf[s][u][1][k]));
                    } else {
                        const double xn = add(buf[s][u][2][k], mul(A.alpha, buf[s][u][0][k]));
                        const double rn = sub(buf[s][u][3][k], mul(A.alpha, buf[s][u][1][k]));
                        st_stream(A.x + off + k, xn);
                        st_stream(A.r + off + k, rn);
                        acc[j] = add(acc[j], mul(rn, rn));
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == ST) {
                s = 0;
                ph ^= 1u;
            }
        }
        // leftover full chunks (< SPS) and the partial last chunk, from global
        // memory, still in chain order
        for (int64_t off = nstage * SPS * S + base0; off < n; off += S) {
#pragma unroll
            for (int j = 0; j < SPT; j++) {
                const int64_t i = off + tid + j * T;
                if (i < n) {
                    Step<MODE> st;
                    st.load(A, i);
                    acc[j] = add(acc[j], step_term<MODE>(st, A, i));
                }
            }
        }
    }
    if (tid < T) {
#pragma unroll
        for (int j = 0; j < SPT; j++) sm[tid + j * T] = acc[j];
    }
    __syncthreads();
    // tree fold of each of the CTA's BPC lattice blocks (LB slots each):
    // threads >= T skip the smem levels; warp h does block h's shuffles
    constexpr int LB = BS / BPC;
    for (int k = LB / 2; k >= 32; k >>= 1) {
        for (int s = tid; s < BPC * k && tid < T; s += T) {  // (the producer warp has tid >= T)
            const int h = s / k, i = s - h * k;
            sm[h * LB + i] = add(sm[h * LB + i], sm[h * LB + i + k]);
        }
        __syncthreads();
    }
    // block values: CTA 0 keeps its own in shared memory, every other CTA
    // publishes them as flagged slots (ll_put, see second_stage)
    __shared__ double own[BPC];
    double v = 0.0;
    if (warp < BPC) {
        constexpr int W = LB < 32 ? LB : 32;
        if (lane < W) v = sm[warp * LB + lane];
        for (int off = W / 2; off >= 1; off >>= 1) v = add(v, __shfl_down_sync(0xffffffffu, v, off));
        if (lane == 0) {
            if (blockIdx.x == 0)
                own[warp] = v;
            else
                ll_put(A.ll + 2 * ((int64_t)blockIdx.x * BPC + warp), v);
        }
    }
    if (blockIdx.x != 0) return;
    __syncthreads();
    // second stage in CTA 0, straight from the flagged slots; consumer threads
    // only (the producer warp, tid >= T, would take slots t >= T twice, and a
    // taken slot is re-zeroed, so the second taker would spin forever)
    for (int t = tid; t < LB && tid < T; t += T) {
        double a2 = 0.0;
        for (int64_t c = t; c < A.nb; c += LB) a2 = add(a2, c < BPC ? own[c] : ll_take(A.ll + 2 * c));
        sm[t] = a2;
    }
    __syncthreads();
    for (int k = LB / 2; k >= 32; k >>= 1) {
        for (int s = tid; s < k && tid < T; s += T) sm[s] = add(sm[s], sm[s + k]);
        __syncthreads();
    }
    if (tid < 32) {
        constexpr int W = LB < 32 ? LB : 32;
        double r = tid < W ? sm[tid] : 0.0;
        for (int off = W / 2; off >= 1; off >>= 1) r = add(r, __shfl_down_sync(0xffffffffu, r, off));
        if (tid == 0) write_result(A, r);
    }
}

// ---- generic path (block_size > 1024): lattice in global memory ----------
template <int MODE>
__global__ void __launch_bounds__(256) k_lattice_global(RArgs Ain) {
    RArgs A = Ain;
    if (!resolve(A)) return;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < A.S;
         s += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int64_t i = s; i < A.n; i += A.S) {
            Step<MODE> st;
            st.load(A, i);
            acc = add(acc, step_term<MODE>(st, A, i));
        }
        A.lattice[s] = acc;
    }
}

// Fold one lattice row (length bs, in global memory) in place; 1024 threads.
__device__ double fold_global_row(double *row, int64_t bs) {
    for (int64_t k = bs / 2; k > 1; k >>= 1) {
        for (int64_t s = threadIdx.x; s < k; s += blockDim.x) row[s] = add(row[s], row[s + k]);
        __syncthreads();
    }
    return add(row[0], row[1]);
}

__global__ void __launch_bounds__(1024) k_fold_blocks(RArgs A) {
    if (A.gate && *A.gate == 0) return;
    const double v = fold_global_row(A.lattice + (int64_t)blockIdx.x * A.bs, A.bs);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = v;
}

__global__ void __launch_bounds__(1024) k_final_generic(RArgs A) {
    if (A.gate && *A.gate == 0) return;
    double *srow = A.lattice + A.S;  // bs scratch doubles
    for (int64_t t = threadIdx.x; t < A.bs; t += blockDim.x) {
        double acc = 0.0;
        for (int64_t c = t; c < A.nb; c += A.bs) acc = add(acc, A.partials[c]);
        srow[t] = acc;
    }
    __syncthreads();
    const double v = fold_global_row(srow, A.bs);
    if (threadIdx.x == 0) write_result(A, v);
}

// block_size 512 halves the steps per stage (same stage bytes)
constexpr int ring_sps(int sps, int bs) { return bs <= 256 ? sps : (sps / 2 > 0 ? sps / 2 : 1); }
constexpr int ring_stages(int ring, int stage_bytes) {
    return ring / stage_bytes > 16 ? 16 : (ring / stage_bytes < 2 ? 2 : ring / stage_bytes);
}

// SB200_NO_TMA=1 selects the register-unrolled lattice kernel (A/B checks).
static bool use_tma() {
    static const bool on = [] {
        const char *e = getenv("SB200_NO_TMA");
        return !(e && e[0] == '1');
    }();
    return on;
}

// SB200_TMA_MIN=<n> moves every mode's register/TMA crossover to n elements
// (tests drive the TMA ring at ragged sizes below the default crossovers).
static int64_t tma_min_override() {
    static const int64_t v = [] {
        const char *e = getenv("SB200_TMA_MIN");
        return e && e[0] ? (int64_t)atoll(e) : (int64_t)-1;
    }();
    return v;
}

// SB200_POLL_LIMIT -> g_sb_poll_limit, once per device (max 64 devices tracked)
static void set_poll_limit_once() {
    static const char *e = getenv("SB200_POLL_LIMIT");
    if (!e || !e[0]) return;
    static unsigned long long done = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || (done >> dev) & 1ull) return;
    const unsigned long long v = strtoull(e, nullptr, 10);
    if (cudaMemcpyToSymbol(g_sb_poll_limit, &v, sizeof(v)) == cudaSuccess) done |= 1ull << dev;
}

template <int MODE>
static int launch_reduce(RArgs A, void *ws, cudaStream_t st, const char *name) {
    clear_error();
    set_poll_limit_once();
    if (A.bs < 2 || (A.bs & (A.bs - 1)) || A.nb < 1) {
        set_error("%s: block_size must be a power of two >= 2 and n_blocks >= 1 (got %lld, %lld)",
                  name, (long long)A.bs, (long long)A.nb);
        return SB_E_INVALID;
    }
    if (A.n < 0 || ws == nullptr || A.result == nullptr || A.nb > 0x7fffffffLL) {
        set_error("%s: invalid arguments", name);
        return SB_E_INVALID;
    }
    char *w = static_cast<char *>(ws);
    A.partials = reinterpret_cast<double *>(w + 256);
    A.ll = reinterpret_cast<unsigned long long *>(w + ll_offset(A.nb));
    A.S = A.bs * A.nb;
    const unsigned grid = (unsigned)A.nb;
    // U (chain unroll) is chosen so the batch keeps >= ~128 B in flight per
    // thread while staying under 64 registers (4 CTAs of 256 per SM).
    constexpr int UN = 16, UD = 8, UF = 4;
    constexpr int U = MODE == R_NORM ? UN : (MODE == R_DOT ? UD : UF);
    // TMA ring: ~32 KB of stages per CTA (so <= 4 CTAs/SM by shared memory)
    constexpr int NA = NArr<MODE>::v;
    const bool tma_ok = aligned16(A.u) && aligned16(A.v) && (MODE != R_FUSED || (aligned16(A.x) && aligned16(A.r)));
    // Register-pipelined lattice below these sizes, TMA ring above: measured
    // crossovers with L2 flushed before every timed batch (graph timer,
    // scripts/expt/run_lat_small.py, profiles/r01_lattice_latency.md) -- BS3
    // ~48M, BS4 ~16M, BS5 ~3M elements.  Same lattice, bitwise the same
    // scalar either way.
#ifndef SB_TMA_MIN_FUSED
#define SB_TMA_MIN_FUSED 3000000
#define SB_TMA_MIN_DOT 16000000
#define SB_TMA_MIN_NORM 48000000
#endif
    constexpr int64_t kTmaMinN =
        MODE == R_FUSED ? SB_TMA_MIN_FUSED : (MODE == R_DOT ? SB_TMA_MIN_DOT : SB_TMA_MIN_NORM);
    const int64_t tma_min = tma_min_override() >= 0 ? tma_min_override() : kTmaMinN;
    if (tma_ok && use_tma() && A.n >= tma_min && (A.bs == 64 || A.bs == 128 || A.bs == 256 || A.bs == 512)) {
        // ring shape (stages x steps per stage): ~32-48 KB of stages per CTA
        constexpr int SPS = MODE == R_NORM ? kSpsNorm : (MODE == R_DOT ? kSpsDot : kSpsFused);
        constexpr int RING = MODE == R_NORM ? kRingNorm : (MODE == R_DOT ? kRingDot : kRingFused);
#define SB_TMA_BR(T_, SPT_, BPC_, RING_)                                                                  \
    {                                                                                                     \
        constexpr int SPS_ = ring_sps(SPS, T_ * SPT_);                                                   \
        constexpr int STB_ = SPS_ * NA * T_ * SPT_ * 8;                                                  \
        constexpr int ST_ = ring_stages(RING_, STB_);                                                     \
        auto kern = k_lattice_tma<T_, SPT_, MODE, ST_, SPS_, BPC_>;                                       \
        static int attr_dev = -1; /* per instantiation and device */                                      \
        int dev = 0;                                                                                      \
        cudaGetDevice(&dev);                                                                              \
        if (attr_dev != dev) {                                                                            \
            if (int rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                                         ST_ * STB_),                                     \
                                    name))                                                                \
                return rc;                                                                                \
            attr_dev = dev;                                                                               \
        }                                                                                                 \
        kern<<<grid / BPC_, T_ + 32, ST_ * STB_, st>>>(A);                                                \
    }
#define SB_TMA_B(T_, SPT_, BPC_) SB_TMA_BR(T_, SPT_, BPC_, RING)
#define SB_TMA(T_, SPT_) SB_TMA_B(T_, SPT_, 1)
        switch (A.bs) {
            case 64: SB_TMA(64, 1); break;
            case 128: SB_TMA(128, 1); break;
            case 256:
                // BS5: four lattice blocks per CTA (8 KB chunks per array per step,
                // one 128 KB ring per SM) -- +4-5% over one block per CTA, whose 2 KB
                // chunks write back less efficiently (profiles/r01_lattice_variants.md);
                // BS3/BS4 (read-only) keep one block per CTA.
                if (MODE == R_FUSED && (A.nb & 3) == 0) SB_TMA_BR(256, 4, 4, kRingFusedBpc4)
                else if (kBpc == 2 && (A.nb & 1) == 0) SB_TMA_B(256, 2, 2)
                else SB_TMA(256, 1);
                break;
            default: SB_TMA(256, 2); break;
        }
#undef SB_TMA_B
#undef SB_TMA_BR
#undef SB_TMA
        return launch_check(name);
    }
    // For n < S every lattice block past ceil(n / bs) is empty: its slots
    // stay +0.0, its tree gives +0.0, and adding +0.0 in the final reduce
    // leaves any running sum (which starts at +0.0 and so is never -0.0)
    // unchanged -- launching only the non-empty blocks is bitwise the same
    // and cuts the small-n fixed cost (fewer partials for CTA 0 to collect).
    const unsigned grid_lat = A.n < A.S ? (unsigned)std::max<int64_t>(1, (A.n + A.bs - 1) / A.bs) : grid;
#define SB_LAT(T_, SPT_) k_lattice<T_, SPT_, MODE, (U / SPT_ > 0 ? U / SPT_ : 1)><<<grid_lat, T_, 0, st>>>(A)  /* same bytes in flight per thread */
    switch (A.bs) {
        case 2: SB_LAT(2, 1); break;
        case 4: SB_LAT(4, 1); break;
        case 8: SB_LAT(8, 1); break;
        case 16: SB_LAT(16, 1); break;
        case 32: SB_LAT(32, 1); break;
        case 64: SB_LAT(64, 1); break;
        case 128: SB_LAT(128, 1); break;
        case 256: SB_LAT(256, 1); break;
        case 512: SB_LAT(256, 2); break;
        case 1024: SB_LAT(256, 4); break;
        default: {
            A.lattice = reinterpret_cast<double *>(w + ll_offset(A.nb) + 16 * (size_t)A.nb);
            const int64_t want = (A.S + 255) / 256;
            const unsigned g = (unsigned)std::min<int64_t>(want, (int64_t)sm_count() * 8);
            k_lattice_global<MODE><<<g, 256, 0, st>>>(A);
            if (int rc = launch_check(name)) return rc;
            k_fold_blocks<<<grid, 1024, 0, st>>>(A);
            if (int rc = launch_check(name)) return rc;
            k_final_generic<<<1, 1024, 0, st>>>(A);
        }
    }
#undef SB_LAT
    return launch_check(name);
}

int cg_reduce(int mode, const double *u, const double *v, double *x, double *r, int64_t n, int64_t bs,
              int64_t nb, void *ws, double *result, const int32_t *gate, const double *alpha,
              cudaStream_t st, const char *name, const LsaArgs *lsa) {
    RArgs A{};
    A.u = u; A.v = v; A.x = x; A.r = r; A.n = n; A.bs = bs; A.nb = nb; A.result = result;
    A.gate = gate; A.alpha_ptr = alpha;
    if (lsa) A.lsa = *lsa;
    if (!gate || (n > 0 && (!u || !v || (mode == R_FUSED && (!x || !r || !alpha))))) {
        set_error("%s: invalid arguments", name);
        return SB_E_INVALID;
    }
    switch (mode) {
        case R_NORM: return launch_reduce<R_NORM>(A, ws, st, name);
        case R_DOT: return launch_reduce<R_DOT>(A, ws, st, name);
        default: return launch_reduce<R_FUSED>(A, ws, st, name);
    }
}

int lsa_reduce(int mode, double alpha, const double *u, const double *v, double *x, double *r, int64_t n,
               int64_t bs, int64_t nb, void *ws, double *result, const LsaArgs &lsa, cudaStream_t st,
               const char *name) {
    RArgs A{};
    A.u = u; A.v = v; A.x = x; A.r = r; A.alpha = alpha; A.n = n; A.bs = bs; A.nb = nb; A.result = result;
    A.lsa = lsa;
    if (n > 0 && (!u || !v || (mode == R_FUSED && (!x || !r)))) {
        set_error("%s: invalid arguments", name);
        return SB_E_INVALID;
    }
    switch (mode) {
        case R_NORM: return launch_reduce<R_NORM>(A, ws, st, name);
        case R_DOT: return launch_reduce<R_DOT>(A, ws, st, name);
        default: return launch_reduce<R_FUSED>(A, ws, st, name);
    }
}

// ---- validators / helpers ------------------------------------------------

__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
    s = add(a, b);
    const double bb = sub(s, a);
    e = add(sub(a, sub(s, bb)), sub(b, bb));
}
__device__ __forceinline__ void dd_add(double &hi, double &lo, double h2, double l2) {
    double s, e;
    two_sum(hi, h2, s, e);
    e = add(e, add(lo, l2));
    two_sum(s, e, hi, lo);
}

__global__ void __launch_bounds__(256) k_dot_dd(const double *u, const double *v, int64_t n, double *hi_p,
                                               double *lo_p, unsigned *ticket, double *result) {
    double hi = 0.0, lo = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s, e;
        two_sum(hi, mul(u[i], v[i]), s, e);
        hi = s;
        lo = add(lo, e);
    }
    __shared__ double sh[256], sl[256];
    sh[threadIdx.x] = hi;
    sl[threadIdx.x] = lo;
    __syncthreads();
    for (int k = 128; k >= 1; k >>= 1) {
        if ((int)threadIdx.x < k) {
            double h = sh[threadIdx.x], l = sl[threadIdx.x];
            dd_add(h, l, sh[threadIdx.x + k], sl[threadIdx.x + k]);
            sh[threadIdx.x] = h;
            sl[threadIdx.x] = l;
        }
        __syncthreads();
    }
    __shared__ bool is_last;
    if (threadIdx.x == 0) {
        hi_p[blockIdx.x] = sh[0];
        lo_p[blockIdx.x] = sl[0];
        __threadfence();
        is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last && threadIdx.x == 0) {
        __threadfence();
        double h = 0.0, l = 0.0;
        for (unsigned b = 0; b < gridDim.x; b++) dd_add(h, l, __ldcg(hi_p + b), __ldcg(lo_p + b));
        *result = add(h, l);
        *ticket = 0u;
    }
}

__global__ void k_sum_ordered(const double *v, int64_t count, double *out) {
    double acc = 0.0;
    for (int64_t i = 0; i < count; i++) acc = add(acc, v[i]);
    *out = acc;
}

}  // namespace sb

using namespace sb;

extern "C" {

size_t sb_reduce_workspace_bytes(int64_t block_size, int64_t n_blocks) {
    if (block_size < 2 || (block_size & (block_size - 1)) || n_blocks < 1) return 0;
    return ws_bytes(block_size, n_blocks);
}

int sb_bs3_norm2(const double *x, int64_t n, int64_t bs, int64_t nb, void *ws, double *result,
                 sb_stream_t s) {
    RArgs A{};
    A.u = x; A.v = x; A.n = n; A.bs = bs; A.nb = nb; A.result = result;
    if (n > 0 && !x) { set_error("sb_bs3_norm2: null x"); return SB_E_INVALID; }
    return launch_reduce<R_NORM>(A, ws, as_stream(s), "sb_bs3_norm2");
}

int sb_bs4_dot(const double *x, const double *y, int64_t n, int64_t bs, int64_t nb, void *ws,
               double *result, sb_stream_t s) {
    RArgs A{};
    A.u = x; A.v = y; A.n = n; A.bs = bs; A.nb = nb; A.result = result;
    if (n > 0 && (!x || !y)) { set_error("sb_bs4_dot: null input"); return SB_E_INVALID; }
    return launch_reduce<R_DOT>(A, ws, as_stream(s), "sb_bs4_dot");
}

int sb_bs5_fused_cg_update(double alpha, const double *p, const double *ap, double *x, double *r,
                           int64_t n, int64_t bs, int64_t nb, void *ws, double *result,
                           sb_stream_t s) {
    RArgs A{};
    A.u = p; A.v = ap; A.x = x; A.r = r; A.alpha = alpha; A.n = n; A.bs = bs; A.nb = nb;
    A.result = result;
    if (n > 0 && (!p || !ap || !x || !r)) {
        set_error("sb_bs5_fused_cg_update: null input");
        return SB_E_INVALID;
    }
    return launch_reduce<R_FUSED>(A, ws, as_stream(s), "sb_bs5_fused_cg_update");
}

int sb_sum_ordered(const double *values, int64_t count, double *result, sb_stream_t s) {
    clear_error();
    if (count < 0 || !result || (count > 0 && !values)) {
        set_error("sb_sum_ordered: invalid arguments");
        return SB_E_INVALID;
    }
    k_sum_ordered<<<1, 1, 0, as_stream(s)>>>(values, count, result);
    return launch_check("sb_sum_ordered");
}

int sb_dot_compensated(const double *u, const double *v, int64_t n, void *ws, double *result,
                       sb_stream_t s) {
    clear_error();
    if (n < 0 || !ws || !result || (n > 0 && (!u || !v))) {
        set_error("sb_dot_compensated: invalid arguments");
        return SB_E_INVALID;
    }
    constexpr int G = 592;  // needs sb_reduce_workspace_bytes(256, 592) = 256 + 592*8 ... x2 below
    char *w = static_cast<char *>(ws);
    unsigned *ticket = reinterpret_cast<unsigned *>(w);
    double *hi = reinterpret_cast<double *>(w + 256);
    double *lo = hi + G / 2;  // G/2 doubles each: grid below uses G/2 CTAs
    k_dot_dd<<<G / 2, 256, 0, as_stream(s)>>>(u, v, n, hi, lo, ticket, result);
    return launch_check("sb_dot_compensated");
}

}  // extern "C"
