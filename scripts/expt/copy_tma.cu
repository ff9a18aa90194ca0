// Probe: BS1 copy through TMA bulk copies (global -> smem -> global) vs the
// LDG/STG stream kernel.  One elected thread per CTA runs a ring of ST
// stages: load chunk i, and store chunk i-LAG once its load has landed.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CH, int ST, int LAG>
__global__ void __launch_bounds__(32) k_copy_tma(const char *x, char *y, int64_t nchunks) {
    extern __shared__ __align__(128) char sbuf[];
    __shared__ __align__(8) uint64_t full[ST];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < ST; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t ph[ST];
    for (int s = 0; s < ST; s++) ph[s] = 0;
    const int64_t g = gridDim.x;
    int64_t k = 0;  // local chunk counter
    for (int64_t c = blockIdx.x;; c += g, k++) {
        const bool load = c < nchunks;
        // store chunk k-LAG (its load was issued LAG iterations ago)
        if (k >= LAG) {
            const int64_t cs = c - (int64_t)LAG * g;
            if (cs < nchunks) {
                const int s = (int)((k - LAG) % ST);
                asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                             ::"r"(su32(&full[s])), "r"(ph[s]) : "memory");
                ph[s] ^= 1;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(y + cs * CH), "r"(su32(sbuf + s * CH)), "r"(CH) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            } else if (!load) {
                break;
            }
        } else if (!load) {
            break;
        }
        if (load) {
            const int s = (int)(k % ST);
            // the stage's previous occupant (chunk k-ST) must have been read by its store
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(ST - LAG - 1) : "memory");
            asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}"
                         ::"r"(su32(&full[s])), "r"(CH) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(sbuf + s * CH)), "l"(x + c * CH), "r"(CH), "r"(su32(&full[s])) : "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

extern "C" int copy_tma(int variant, const void *x, void *y, int64_t bytes, int grid, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
#define RUN(CH, ST, LAG)                                                                                     \
    {                                                                                                        \
        auto k = k_copy_tma<CH, ST, LAG>;                                                                   \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST);                      \
        k<<<grid, 32, CH * ST, st>>>((const char *)x, (char *)y, bytes / CH);                               \
    }
    switch (variant) {
        case 0: RUN(16384, 8, 4); break;
        case 1: RUN(32768, 6, 3); break;
        case 2: RUN(8192, 16, 8); break;
        default: RUN(16384, 12, 6); break;
    }
#undef RUN
    return (int)cudaGetLastError();
}
