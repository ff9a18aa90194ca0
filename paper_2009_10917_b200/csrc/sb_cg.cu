// sb_cg.cu -- device-resident Conjugate Gradient steps (cg.py:27-72 with the
// scalars kept on the GPU).
//
// The reference pulls p.Ap and r.r to the host every iteration (two syncs)
// to form alpha = rr / pAp and beta = rr_new / rr.  Here those scalars live
// in an sb_cg_state in device memory and the kernels read them at entry:
//   sb_cg_pap        BS4 lattice dot -> st->pap, then the SPD check and
//                    alpha = rr / pap (one-thread control kernel)
//   sb_cg_update     fused BS5 with alpha read from st -> st->rr_new, or the
//                    unfused BS2, BS2, BS3 sequence (bitwise the same)
//   sb_cg_direction  beta = rr_new / rr; p = 1.0*r + beta*p (BS2); then
//                    rr = rr_new, iterations += 1,
//                    active = rr > tol && iterations < max_iter
// Every kernel is gated on st->active, so once the solve has converged (or
// hit max_iter, or met p.Ap <= 0) further launched iterations do nothing and
// the host needs to look at the state only once per batch of iterations
// (one small D2H read; the batch can be a captured CUDA graph).  The
// divisions are IEEE correctly rounded like Python's, so iterates, iteration
// count and final r.r are bitwise those of the host-scalar solver.
#include "sb_common.cuh"

namespace sb {

__global__ void k_cg_begin(sb_cg_state *st, const double *rr0, const double *bb, double eps, int64_t max_iter) {
    const double rr = *rr0;
    const double tol = bb ? __dmul_rn(eps, *bb) : eps;
    st->rr = rr;
    st->rr_new = 0.0;
    st->pap = 0.0;
    st->tol = tol;
    st->iterations = 0;
    st->max_iter = max_iter;
    st->fail_pap = 0.0;
    st->alpha = 0.0;
    st->beta = 0.0;
    st->status = SB_CG_RUNNING;
    // cg.py:58: while rr > tol and iterations < max_iter
    st->active = (rr > tol && max_iter > 0) ? 1 : 0;
    if (!st->active) st->status = rr > tol ? SB_CG_EXHAUSTED : SB_CG_CONVERGED;
}

// cg.py:61-65: raise NotSPDError if p.Ap <= 0.0 (a NaN passes, as in
// Python), else alpha = rr / pAp
__global__ void k_cg_check(sb_cg_state *st) {
    if (!st->active) return;
    if (st->pap <= 0.0) {
        st->active = 0;
        st->status = SB_CG_NOT_SPD;
        st->fail_pap = st->pap;
        return;
    }
    st->alpha = __ddiv_rn(st->rr, st->pap);
}

// cg.py:70: beta = rr_new / rr
__global__ void k_cg_beta(sb_cg_state *st) {
    if (!st->active) return;
    st->beta = __ddiv_rn(st->rr_new, st->rr);
}

__global__ void k_cg_advance(sb_cg_state *st) {
    if (!st->active) return;
    st->rr = st->rr_new;
    st->iterations += 1;
    if (!(st->rr > st->tol)) {
        st->active = 0;
        st->status = SB_CG_CONVERGED;
    } else if (st->iterations >= st->max_iter) {
        st->active = 0;
        st->status = SB_CG_EXHAUSTED;
    }
}

int cg_pap_impl(const double *p, const double *ap, int64_t n, int64_t bs, int64_t nb, void *ws,
                sb_cg_state *st, const LsaArgs *lsa, cudaStream_t cs) {
    if (!st) {
        set_error("sb_cg_pap: null state");
        return SB_E_INVALID;
    }
    if (int rc = cg_reduce(1, p, ap, nullptr, nullptr, n, bs, nb, ws, &st->pap, &st->active, nullptr, cs,
                           "sb_cg_pap", lsa))
        return rc;
    k_cg_check<<<1, 1, 0, cs>>>(st);
    return launch_check("sb_cg_pap");
}

int cg_update_impl(int fused, const double *p, const double *ap, double *x, double *r, int64_t n, int64_t bs,
                   int64_t nb, void *ws, sb_cg_state *st, const LsaArgs *lsa, cudaStream_t cs) {
    if (!st) {
        set_error("sb_cg_update: null state");
        return SB_E_INVALID;
    }
    if (fused)  // kernels.py:117-132 with alpha from the state
        return cg_reduce(2, p, ap, x, r, n, bs, nb, ws, &st->rr_new, &st->active, &st->alpha, cs,
                         "sb_cg_update", lsa);
    // cg.py:67-70: x = alpha*p + 1.0*x ; r = (-alpha)*ap + 1.0*r ; rr_new = r.r
    const DevCoef alpha{&st->alpha, 1.0}, neg_alpha{&st->alpha, -1.0}, one{nullptr, 1.0};
    if (int rc = cg_axpy(p, x, n, alpha, one, &st->active, cs, "sb_cg_update")) return rc;
    if (int rc = cg_axpy(ap, r, n, neg_alpha, one, &st->active, cs, "sb_cg_update")) return rc;
    return cg_reduce(0, r, r, nullptr, nullptr, n, bs, nb, ws, &st->rr_new, &st->active, nullptr, cs,
                     "sb_cg_update", lsa);
}

}  // namespace sb

using namespace sb;

extern "C" {

int sb_cg_begin(sb_cg_state *st, const double *rr0, const double *bb, double eps, int64_t max_iter,
                sb_stream_t s) {
    clear_error();
    if (!st || !rr0 || eps <= 0.0 || max_iter < 0) {  // cg.py:40-41 (a NaN eps passes, as in Python)
        set_error("sb_cg_begin: invalid arguments (eps must be positive)");
        return SB_E_INVALID;
    }
    k_cg_begin<<<1, 1, 0, as_stream(s)>>>(st, rr0, bb, eps, max_iter);
    return launch_check("sb_cg_begin");
}

int sb_cg_pap(const double *p, const double *ap, int64_t n, int64_t bs, int64_t nb, void *ws, sb_cg_state *st,
              sb_stream_t s) {
    clear_error();
    return cg_pap_impl(p, ap, n, bs, nb, ws, st, nullptr, as_stream(s));
}

int sb_cg_update(int fused, const double *p, const double *ap, double *x, double *r, int64_t n, int64_t bs,
                 int64_t nb, void *ws, sb_cg_state *st, sb_stream_t s) {
    clear_error();
    return cg_update_impl(fused, p, ap, x, r, n, bs, nb, ws, st, nullptr, as_stream(s));
}

int sb_cg_direction(const double *r, double *p, int64_t n, sb_cg_state *st, sb_stream_t s) {
    clear_error();
    if (!st) {
        set_error("sb_cg_direction: null state");
        return SB_E_INVALID;
    }
    // cg.py:70-71: beta = rr_new / rr ; p = 1.0*r + beta*p
    k_cg_beta<<<1, 1, 0, as_stream(s)>>>(st);
    if (int rc = launch_check("sb_cg_direction")) return rc;
    const DevCoef one{nullptr, 1.0}, beta{&st->beta, 1.0};
    if (int rc = cg_axpy(r, p, n, one, beta, &st->active, as_stream(s), "sb_cg_direction")) return rc;
    k_cg_advance<<<1, 1, 0, as_stream(s)>>>(st);
    return launch_check("sb_cg_direction");
}

}  // extern "C"
