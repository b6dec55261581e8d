// Device Krylov drivers around the preconditioner: deterministic fused
// BLAS-1 reductions, BiCGSTAB (the contract defined in oracle/iluk_oracle.py)
// and restarted GMRES(m) with left preconditioning (gmres.py:76-186).
//
// Every reduction is two-pass with a FIXED partition (RED_BLOCKS blocks of
// RED_THREADS threads, contiguous chunks, fixed shared-memory tree), so the
// results are bitwise repeatable run to run, independent of the GPU.
// Scalars (alpha, omega, rho, beta, H entries) live on the device; the host
// reads back only what its stopping tests need.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "biluk_internal.h"
#include "device_util.cuh"
#include "kernels.cuh"

namespace biluk {

constexpr int RED_BLOCKS = 512;
constexpr int RED_THREADS = 256;
constexpr int MAXQ = 3;
constexpr int64_t HIST_CAP = 65536;   // device residual-history entries kept in a Krylov workspace


// scalar slots in DevStatus::scal
enum {
    S_RHO = 0, S_RHO_PREV, S_ALPHA, S_OMEGA, S_BETA, S_RV, S_SS, S_TT, S_TS, S_RR, S_RHO_NEXT, S_GEN0, S_GEN1,
    S_GEN2, S_HPREV, S_H0 = 16,  // S_H0.. : scratch for the current GMRES column
    // batched BiCGSTAB (per-system block of B_STRIDE slots; S_H0.. unused there)
    S_BN = 16, S_XA, S_XW, S_ITS, S_NH, S_LAST, S_TRUE, B_STRIDE = 24
};

__device__ __forceinline__ double block_sum(double v, double *sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
#pragma unroll
    for (int w = RED_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// Fused elementwise update + up to three dot products, one pass:
//   op 0: out = a . b                                   (dots only)
//   op 1: u = x + c0 * v                ; dots over updated u  (axpy)
//   op 2: u = x + c0 * (u - c1 * v)     (BiCGSTAB p update, no dots)
//   op 3: u = u + c0 * v + c1 * w       (x update)
// coefficients come from device scalar slots (negative index = constant 0).
struct Fused {
    int op;
    double *u;
    const double *v, *w, *x;
    int ic0, ic1;      // scalar slot indices
    double sgn0;       // multiplies c0 (lets one slot serve +alpha and -alpha)
    int nq;
    const double *qa[MAXQ];
    const double *qb[MAXQ];   // dot q: qa[q] . qb[q]; nullptr means "the updated u"
};

// Batched form (independent systems packed back to back, biluk_bicgstab_batched):
// block sys * RED_BLOCKS + j reduces chunk j of system sys's segment
// [seg[sys], seg[sys+1]) -- the same partition a single solve of that system
// uses, so a system's reductions round as in its own solve.  `state`
// gates the update per system (skipped when state[sys] > smax).
struct Batch {
    const int64_t *seg;   // nullptr: one system [0, len)
    const int *state;
    int smax;
    int sstride;          // scalar slots per system
};

__global__ void __launch_bounds__(RED_THREADS) fused_kernel(Fused f, int64_t len, const double *scal, double *partials,
                                                            const int *skip, Batch bt) {
    __shared__ double sh[RED_THREADS];
    if (skip && *skip) return;
    const int sys = blockIdx.x / RED_BLOCKS;
    const int blk = blockIdx.x % RED_BLOCKS;
    if (bt.state && bt.state[sys] > bt.smax) return;
    const int64_t base = bt.seg ? bt.seg[sys] : 0;
    const int64_t slen = bt.seg ? bt.seg[sys + 1] - base : len;
    scal += int64_t(sys) * bt.sstride;
    partials += int64_t(sys) * MAXQ * RED_BLOCKS;
    const double c0 = f.ic0 >= 0 ? f.sgn0 * scal[f.ic0] : 0.0;
    const double c1 = f.ic1 >= 0 ? scal[f.ic1] : 0.0;
    const int64_t chunk = (slen + RED_BLOCKS - 1) / RED_BLOCKS;
    const int64_t lo = base + int64_t(blk) * chunk;
    const int64_t hi = lo + chunk < base + slen ? lo + chunk : base + slen;
    double acc[MAXQ] = {0.0, 0.0, 0.0};
    for (int64_t i = lo + threadIdx.x; i < hi; i += RED_THREADS) {
        double uval = 0.0;
        switch (f.op) {
            case 1: uval = f.x[i] + c0 * f.v[i]; f.u[i] = uval; break;
            case 2: uval = f.x[i] + c0 * (f.u[i] - c1 * f.v[i]); f.u[i] = uval; break;
            case 3: uval = f.u[i] + c0 * f.v[i] + c1 * f.w[i]; f.u[i] = uval; break;
            default: break;
        }
#pragma unroll
        for (int q = 0; q < MAXQ; ++q)
            if (q < f.nq) {
                const double a = f.qa[q] ? f.qa[q][i] : uval;
                const double b = f.qb[q] ? f.qb[q][i] : uval;
                acc[q] = fma(a, b, acc[q]);
            }
    }
    for (int q = 0; q < f.nq; ++q) {
        const double s = block_sum(acc[q], sh);
        if (threadIdx.x == 0) partials[q * RED_BLOCKS + blk] = s;
    }
}

// Second pass: sum the partials of nq dots in fixed order into scal[dst[q]],
// then run the scalar epilogue `op`.  One block per system.
enum { FIN_NONE = 0, FIN_ALPHA, FIN_OMEGA, FIN_BETA, FIN_DIV, FIN_GMRES_H,
       FIN_B_INIT, FIN_B_ALPHA, FIN_B_HALF, FIN_B_OMEGA, FIN_B_BETA, FIN_B_TRUE };

// batched per-system state: 0 iterating, 1 finishing (x update pending), 2 stopped
struct BFin {
    int *state;
    double tol;
    int *alive;      // systems not yet stopped; the last one to stop sets *dead
    int *dead;       // every system stopped: the skip word of the apply and SpMV launches
    double *hist;    // one system: its residual history (S_NH entries), or null
    int64_t hcap;
};

__global__ void __launch_bounds__(RED_THREADS) finalize_kernel(const double *partials, int nq, int d0, int d1, int d2,
                                                               int op, double *scal, const int *skip, int sstride,
                                                               BFin bf) {
    __shared__ double sh[RED_THREADS];
    if (skip && *skip) return;
    const int sys = blockIdx.x;
    partials += int64_t(sys) * MAXQ * RED_BLOCKS;
    scal += int64_t(sys) * sstride;
    const int dst[3] = {d0, d1, d2};
    for (int q = 0; q < nq; ++q) {
        double v = 0.0;
        for (int b = threadIdx.x; b < RED_BLOCKS; b += RED_THREADS) v += partials[q * RED_BLOCKS + b];
        const double s = block_sum(v, sh);
        if (threadIdx.x == 0) scal[dst[q]] = s;
    }
    if (threadIdx.x != 0) return;
    int *st = bf.state ? bf.state + sys : nullptr;
    auto stop = [&]() {   // state -> 2 (stopped), once per system
        if (*st == 2) return;
        *st = 2;
        if (bf.alive && atomicSub(bf.alive, 1) == 1) *bf.dead = 1;
    };
    auto record = [&](double v) {   // history entry S_NH, then S_NH += 1
        const int64_t k = int64_t(scal[S_NH]);
        if (bf.hist && k < bf.hcap) bf.hist[k] = v;
        scal[S_NH] += 1.0;
    };
    switch (op) {
        case FIN_ALPHA:   // alpha = rho / <r^, v>
            if (scal[S_RV] != 0.0) scal[S_ALPHA] = scal[S_RHO] / scal[S_RV];
            break;
        case FIN_OMEGA:   // omega = <t, s> / <t, t>
            if (scal[S_TT] != 0.0) scal[S_OMEGA] = scal[S_TS] / scal[S_TT];
            break;
        case FIN_BETA:    // next iteration: beta = (rho_n / rho)(alpha / omega); rho <- rho_n
            scal[S_BETA] = (scal[S_RHO_NEXT] / scal[S_RHO]) * (scal[S_ALPHA] / scal[S_OMEGA]);
            scal[S_RHO_PREV] = scal[S_RHO];
            scal[S_RHO] = scal[S_RHO_NEXT];
            break;
        // ---- batched BiCGSTAB: the host-side tests of biluk_bicgstab, per system ----
        case FIN_B_INIT: {   // S_GEN0 = <b, b>
            const double bb = scal[S_GEN0];
            scal[S_BN] = sqrt(bb);
            scal[S_RHO] = bb; scal[S_RHO_PREV] = 1.0; scal[S_ALPHA] = 1.0; scal[S_OMEGA] = 1.0; scal[S_BETA] = bb;
            scal[S_ITS] = 0.0; scal[S_NH] = 0.0; scal[S_LAST] = INFINITY;
            *st = 0;
            if (bb == 0.0) {
                scal[S_LAST] = 0.0;
                stop();
            }
            break;
        }
        case FIN_B_ALPHA:
            if (*st != 0) break;
            if (scal[S_RV] == 0.0) { stop(); break; }   // breakdown before the iteration counts
            scal[S_ALPHA] = scal[S_RHO] / scal[S_RV];
            scal[S_ITS] += 1.0;
            break;
        case FIN_B_HALF: {
            if (*st != 0) break;
            const double sn = sqrt(scal[S_SS]) / scal[S_BN];
            scal[S_LAST] = sn;
            if (sn <= bf.tol) {   // x += alpha p^, stop
                scal[S_XA] = scal[S_ALPHA]; scal[S_XW] = 0.0; record(sn); *st = 1;
            }
            break;
        }
        case FIN_B_OMEGA:
            if (*st != 0) break;
            scal[S_XA] = scal[S_ALPHA];
            if (scal[S_TT] == 0.0) { scal[S_XW] = 0.0; record(scal[S_LAST]); *st = 1; break; }
            scal[S_OMEGA] = scal[S_TS] / scal[S_TT];
            scal[S_XW] = scal[S_OMEGA];
            break;
        case FIN_B_BETA: {
            if (*st == 1) { stop(); break; }
            if (*st != 0) break;
            const double rn = sqrt(scal[S_RR]) / scal[S_BN];
            scal[S_LAST] = rn;
            record(rn);
            const double om = scal[S_OMEGA];
            scal[S_BETA] = (scal[S_RHO_NEXT] / scal[S_RHO]) * (scal[S_ALPHA] / om);
            scal[S_RHO_PREV] = scal[S_RHO];
            scal[S_RHO] = scal[S_RHO_NEXT];
            if (rn <= bf.tol || om == 0.0 || scal[S_RHO] == 0.0) stop();
            break;
        }
        case FIN_B_TRUE:   // S_GEN1 = ||b - A x||^2
            scal[S_TRUE] = scal[S_BN] == 0.0 ? 0.0 : sqrt(scal[S_GEN1]) / scal[S_BN];
            break;
        default: break;
    }
}

// mode 0: c = scal[idx]; 1: c = 1/scal[idx]; 2: c = 1/sqrt(scal[idx])
__global__ void scale_copy_kernel(double *dst, const double *src, int64_t len, const double *scal, int idx, int mode) {
    const double c = mode == 2 ? 1.0 / sqrt(scal[idx]) : (mode == 1 ? 1.0 / scal[idx] : scal[idx]);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = c * src[i];
}

__global__ void combo_kernel(double *x, const double *V, int64_t ld, int64_t len, const double *y, int used) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x) {
        double acc = x[i];
        for (int q = 0; q < used; ++q) acc += V[q * ld + i] * y[q];
        x[i] = acc;
    }
}

__global__ void sub_kernel(double *out, const double *a, const double *b, int64_t len) {   // out = a - b
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < len; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = a[i] - b[i];
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
struct Ctx {
    biluk_op *A;
    biluk_plan *M;
    biluk_precond_fn cb;
    void *user;
    cudaStream_t s;
    int64_t len;
    double *scal;
    double *partials;
    int grid;
    cudaError_t err = cudaSuccess;
    int prc = BILUK_OK;   // the preconditioner's own status when it failed (plan apply or callback)
    // batched solves (biluk_bicgstab_batched); defaults describe one system
    int nsys = 1;
    const int64_t *seg = nullptr;
    int *state = nullptr;
    int smax = 0;
    int sstride = 0;
    double tol = 0.0;
    int *alive = nullptr, *dead = nullptr;   // device liveness words (batched engine)
    double *hist = nullptr;                  // device residual history (one system)
    int64_t hcap = 0;
    const int *skip = nullptr;               // skip word of the SpMV and apply launches

    void fused(const Fused &f) {
        if (err) return;
        fused_kernel<<<RED_BLOCKS * nsys, RED_THREADS, 0, s>>>(f, len, scal, partials, nullptr,
                                                                Batch{seg, state, smax, sstride});
        err = cudaGetLastError();
    }
    void fin(int nq, int d0, int d1, int d2, int op) {
        if (err) return;
        finalize_kernel<<<nsys, RED_THREADS, 0, s>>>(partials, nq, d0, d1, d2, op, scal, nullptr, sstride,
                                                     BFin{state, tol, alive, dead, hist, hcap});
        err = cudaGetLastError();
    }
    void dot(const double *a, const double *b, int dst) {
        Fused f{};
        f.op = 0;
        f.ic0 = f.ic1 = -1;
        f.nq = 1;
        f.qa[0] = a;
        f.qb[0] = b;
        fused(f);
        fin(1, dst, 0, 0, FIN_NONE);
    }
    void spmv(const double *x, double *y) {
        if (err) return;
        err = launch_spmv(A->o, x, y, skip, s);
    }
    int sms() const { return A->o.num_sms; }
    int apply(const double *b, double *x);
    void read(double *host, int idx, int cnt) {
        if (err) return;
        err = cudaMemcpyAsync(host, scal + idx, 8 * cnt, cudaMemcpyDeviceToHost, s);
        if (!err) err = cudaStreamSynchronize(s);
    }
    void set(int idx, double v) {
        if (err) return;
        err = cudaMemcpyAsync(scal + idx, &v, 8, cudaMemcpyHostToDevice, s);
        if (!err) err = cudaStreamSynchronize(s);   // v lives on the host stack
    }
    void copy(double *dst, const double *src) {
        if (err) return;
        err = cudaMemcpyAsync(dst, src, 8 * len, cudaMemcpyDeviceToDevice, s);
    }
    void zero(double *dst) {
        if (err) return;
        err = cudaMemsetAsync(dst, 0, 8 * len, s);
    }
};

}  // namespace biluk

using namespace biluk;

extern "C" int biluk_plan_apply(biluk_plan_t *plan, const double *dev_b, double *dev_x, void *stream);
extern "C" const char *biluk_last_error(void);

// preconditioner: plan apply, else the user callback, else identity
int biluk::Ctx::apply(const double *b, double *x) {
    if (err) return BILUK_ECUDA;
    int rc = BILUK_OK;
    if (M) {
        rc = plan_apply(M, b, x, s, skip);
    } else if (cb) {
        rc = cb(user, b, x, s);
        if (rc != BILUK_OK) fail(rc, "preconditioner callback failed");
    } else {
        err = cudaMemcpyAsync(x, b, 8 * len, cudaMemcpyDeviceToDevice, s);
        return err ? BILUK_ECUDA : BILUK_OK;
    }
    if (rc != BILUK_OK) {
        prc = rc;
        err = cudaErrorUnknown;
    }
    return rc;
}

namespace biluk {
int bicgstab_engine(biluk_op_t *A, biluk_plan_t *M, biluk_precond_fn cb, void *user, int32_t nsys, const int64_t *seg,
                    const double *dev_b, double *dev_x, void *dev_work, int64_t max_iters, double rel_tol,
                    double *stats, double *history, int64_t hist_cap, cudaStream_t stream);
}  // namespace biluk

static int krylov_fail(Ctx &c, const char *what) {
    // the preconditioner already set the message: pass its status on (e.g.
    // BILUK_EARG from a callback that returned a wrong-length vector)
    if (c.err == cudaErrorUnknown) return c.prc != BILUK_OK ? c.prc : BILUK_ECUDA;
    if (c.err != cudaSuccess)
        return fail(BILUK_ECUDA, std::string(what) + ": " + cudaGetErrorString(c.err));
    return BILUK_OK;
}

extern "C" {

uint64_t biluk_krylov_workspace_bytes(int64_t len_, int32_t restart) {
    if (len_ < 0) return 0;
    const uint64_t len = uint64_t(len_);
    const uint64_t vec = ((8 * len + 255) / 256) * 256;
    const uint64_t nvec = 8 + (restart > 0 ? uint64_t(restart) + 1 : 0);
    return nvec * vec + 8 * RED_BLOCKS * MAXQ + 8 * (64 + uint64_t(restart > 0 ? restart : 0) + 2) + 4096 +
           8 * uint64_t(HIST_CAP);
}

int biluk_dot(const double *dev_a, const double *dev_b, int64_t len, double *result, void *dev_work, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double *partials = static_cast<double *>(dev_work);
    double *scal = partials + RED_BLOCKS * MAXQ;
    Fused f{};
    f.op = 0;
    f.ic0 = f.ic1 = -1;
    f.nq = 1;
    f.qa[0] = dev_a;
    f.qb[0] = dev_b;
    fused_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(f, len, scal, partials, nullptr, Batch{nullptr, nullptr, 0, 0});
    finalize_kernel<<<1, RED_THREADS, 0, s>>>(partials, 1, 0, 0, 0, FIN_NONE, scal, nullptr, 0,
                                              BFin{nullptr, 0.0, nullptr, nullptr, nullptr, 0});
    cudaError_t e = cudaMemcpyAsync(result, scal, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(BILUK_ECUDA, std::string("dot: ") + cudaGetErrorString(e));
    return BILUK_OK;
}

// BiCGSTAB, right preconditioned, x0 = 0 -- see oracle/iluk_oracle.py:bicgstab
int biluk_bicgstab(biluk_op_t *A, biluk_plan_t *M, biluk_precond_fn cb, void *user, const double *dev_b,
                   double *dev_x, void *dev_work, int64_t max_iters, double rel_tol, double *stats, double *history,
                   int64_t hist_cap, void *stream) {
    if (!A || !A->o.valued) return fail(BILUK_EARG, "operator has no values");
    if (A->o.n != A->o.ncols) return fail(BILUK_EARG, "bicgstab requires a square matrix");
    if (M && (!M->p.factored || M->p.n * M->p.bs != A->o.n * A->o.bs))   // vectors must match; blockings may differ
        return fail(BILUK_EARG, "preconditioner does not match the operator");
    if (max_iters < 1 || !(rel_tol > 0.0)) return fail(BILUK_EARG, "bad solver configuration");
    if (!cb && !std::getenv("BILUK_KRYLOV_HOST")) {   // device-driven loop (CUDA graph), one system
        const int64_t seg1[2] = {0, A->o.n};
        return bicgstab_engine(A, M, cb, user, 1, seg1, dev_b, dev_x, dev_work, max_iters, rel_tol, stats, history,
                               hist_cap, static_cast<cudaStream_t>(stream));
    }
    const int64_t len = A->o.n * A->o.bs;
    const int32_t precond = (M || cb) ? 1 : 0;
    const uint64_t vec = ((8 * uint64_t(len) + 255) / 256) * 256;
    unsigned char *w = static_cast<unsigned char *>(dev_work);
    double *r = reinterpret_cast<double *>(w + 0 * vec);
    double *rh = reinterpret_cast<double *>(w + 1 * vec);
    double *pv = reinterpret_cast<double *>(w + 2 * vec);
    double *v = reinterpret_cast<double *>(w + 3 * vec);
    double *ph = reinterpret_cast<double *>(w + 4 * vec);
    double *sv = reinterpret_cast<double *>(w + 5 * vec);
    double *sh = reinterpret_cast<double *>(w + 6 * vec);
    double *t = reinterpret_cast<double *>(w + 7 * vec);
    double *partials = reinterpret_cast<double *>(w + 8 * vec);
    double *scal = partials + RED_BLOCKS * MAXQ;
    Ctx c{A, M, cb, user, static_cast<cudaStream_t>(stream), len, scal, partials, 0};
    int64_t nh = 0;
    auto hist = [&](double v) {
        if (history && nh < hist_cap) history[nh] = v;
        ++nh;
    };
    stats[0] = 0;
    stats[1] = 0;
    stats[2] = INFINITY;
    stats[3] = 0;
    c.zero(dev_x);
    c.dot(dev_b, dev_b, S_GEN0);
    double bb = 0;
    c.read(&bb, S_GEN0, 1);
    if (c.err) return krylov_fail(c, "bicgstab");
    const double bnorm = std::sqrt(bb);
    if (len == 0 || bnorm == 0.0) {
        stats[1] = 1;
        stats[2] = 0;
        return BILUK_OK;
    }
    c.copy(r, dev_b);
    c.copy(rh, dev_b);
    c.zero(pv);
    c.zero(v);
    // rho_1 = <r^, r> = <b, b>; rho_prev = alpha = omega = 1  ->  beta_1 = rho_1
    {
        double init[5] = {bb, 1.0, 1.0, 1.0, bb};   // S_RHO, S_RHO_PREV, S_ALPHA, S_OMEGA, S_BETA
        if (!c.err) c.err = cudaMemcpyAsync(scal + S_RHO, init, sizeof(init), cudaMemcpyHostToDevice, c.s);
        if (!c.err) c.err = cudaStreamSynchronize(c.s);
    }
    const double *M_p = precond ? ph : pv;   // unpreconditioned: p^ = p, s^ = s
    const double *M_s = precond ? sh : sv;
    int64_t its = 0;
    double rho = bb;
    for (int64_t it = 1; it <= max_iters; ++it) {
        if (rho == 0.0) break;
        // p = r + beta (p - omega v)
        Fused f{};
        f.op = 2; f.u = pv; f.v = v; f.x = r; f.ic0 = S_BETA; f.ic1 = S_OMEGA; f.sgn0 = 1.0; f.nq = 0;
        c.fused(f);
        if (precond && c.apply(pv, ph) != BILUK_OK) return krylov_fail(c, "bicgstab");
        c.spmv(M_p, v);
        c.dot(rh, v, S_RV);
        c.fin(0, 0, 0, 0, FIN_ALPHA);
        // s = r - alpha v ; ||s||^2
        Fused fs{};
        fs.op = 1; fs.u = sv; fs.x = r; fs.v = v; fs.ic0 = S_ALPHA; fs.ic1 = -1; fs.sgn0 = -1.0; fs.nq = 1;
        fs.qa[0] = nullptr; fs.qb[0] = nullptr;
        c.fused(fs);
        c.fin(1, S_SS, 0, 0, FIN_NONE);
        double chk[2] = {0, 0};   // rv, ss
        c.read(&chk[0], S_RV, 2);
        if (c.err) return krylov_fail(c, "bicgstab");
        if (chk[0] == 0.0) break;
        its = it;
        const double sn = std::sqrt(chk[1]) / bnorm;
        if (sn <= rel_tol) {
            Fused fx{};
            fx.op = 3; fx.u = dev_x; fx.v = M_p; fx.w = M_p; fx.ic0 = S_ALPHA; fx.ic1 = -1; fx.sgn0 = 1.0;
            c.fused(fx);
            hist(sn);
            break;
        }
        if (precond && c.apply(sv, sh) != BILUK_OK) return krylov_fail(c, "bicgstab");
        c.spmv(M_s, t);
        {
            Fused fd{};
            fd.op = 0; fd.ic0 = fd.ic1 = -1; fd.nq = 2;
            fd.qa[0] = t; fd.qb[0] = t; fd.qa[1] = t; fd.qb[1] = sv;
            c.fused(fd);
            c.fin(2, S_TT, S_TS, 0, FIN_OMEGA);
        }
        double tt = 0;
        c.read(&tt, S_TT, 1);
        if (c.err) return krylov_fail(c, "bicgstab");
        if (tt == 0.0) {
            Fused fx{};
            fx.op = 3; fx.u = dev_x; fx.v = M_p; fx.w = M_p; fx.ic0 = S_ALPHA; fx.ic1 = -1; fx.sgn0 = 1.0;
            c.fused(fx);
            hist(sn);
            break;
        }
        // x += alpha p^ + omega s^
        Fused fx{};
        fx.op = 3; fx.u = dev_x; fx.v = M_p; fx.w = M_s; fx.ic0 = S_ALPHA; fx.ic1 = S_OMEGA; fx.sgn0 = 1.0;
        c.fused(fx);
        // r = s - omega t ; ||r||^2 ; rho_next = <r^, r>
        Fused fr{};
        fr.op = 1; fr.u = r; fr.x = sv; fr.v = t; fr.ic0 = S_OMEGA; fr.ic1 = -1; fr.sgn0 = -1.0; fr.nq = 2;
        fr.qa[0] = nullptr; fr.qb[0] = nullptr; fr.qa[1] = rh; fr.qb[1] = nullptr;
        c.fused(fr);
        c.fin(2, S_RR, S_RHO_NEXT, 0, FIN_BETA);
        double sc[8];   // S_OMEGA .. S_RHO_NEXT in one read
        c.read(sc, S_OMEGA, 8);
        if (c.err) return krylov_fail(c, "bicgstab");
        const double om = sc[0];
        const double rn = std::sqrt(sc[S_RR - S_OMEGA]) / bnorm;
        hist(rn);
        rho = sc[S_RHO_NEXT - S_OMEGA];
        if (rn <= rel_tol) break;
        if (om == 0.0) break;
    }
    // true residual ||b - A x|| / ||b||
    c.spmv(dev_x, t);
    if (!c.err) {
        sub_kernel<<<c.sms() * 8, 256, 0, c.s>>>(t, dev_b, t, len);
        c.err = cudaGetLastError();
    }
    c.dot(t, t, S_GEN1);
    double res2 = 0;
    c.read(&res2, S_GEN1, 1);
    if (c.err) return krylov_fail(c, "bicgstab");
    const double rel = std::sqrt(res2) / bnorm;
    stats[0] = double(its);
    stats[1] = rel <= rel_tol ? 1 : 0;
    stats[2] = rel;
    stats[3] = double(nh);
    return M ? biluk_plan_status(M, stream) : BILUK_OK;
}

uint64_t biluk_krylov_batched_workspace_bytes(int64_t len_, int32_t nsys) {
    if (len_ < 0 || nsys < 1) return 0;
    const uint64_t len = uint64_t(len_);
    const uint64_t vec = ((8 * len + 255) / 256) * 256;
    const uint64_t ns = uint64_t(nsys);
    return 8 * vec + 8 * RED_BLOCKS * MAXQ * ns + 8 * B_STRIDE * ns + 8 * (ns + 1) + 4 * ns + 4096 +
           8 * uint64_t(HIST_CAP);
}

// Batched BiCGSTAB: nsys independent systems packed as one block-diagonal
// operator (system s = block rows [seg[s], seg[s+1])) and one preconditioner
// over it.  Every system runs exactly the iteration of biluk_bicgstab on its
// own segment -- its own scalars, stopping tests and iteration count, with the
// same reduction partition as a single solve (x_s equals the single solve's up
// to the rounding of the preconditioner, whose record layout differs in a
// batch) -- while the SpMV and the preconditioner sweeps cover all systems in
// one launch each (their level chains interleave).  A stopped system is frozen;
// the loop ends when every system has stopped.
int biluk_bicgstab_batched(biluk_op_t *A, biluk_plan_t *M, biluk_precond_fn cb, void *user, int32_t nsys,
                           const int64_t *seg, const double *dev_b, double *dev_x, void *dev_work, int64_t max_iters,
                           double rel_tol, double *stats, void *stream) {
    if (!A || !A->o.valued) return fail(BILUK_EARG, "operator has no values");
    if (A->o.n != A->o.ncols) return fail(BILUK_EARG, "bicgstab requires a square matrix");
    if (M && (!M->p.factored || M->p.n * M->p.bs != A->o.n * A->o.bs))   // vectors must match; blockings may differ
        return fail(BILUK_EARG, "preconditioner does not match the operator");
    if (max_iters < 1 || !(rel_tol > 0.0)) return fail(BILUK_EARG, "bad solver configuration");
    if (nsys < 1 || !seg || !stats) return fail(BILUK_EARG, "bad batch description");
    if (seg[0] != 0 || seg[nsys] != A->o.n) return fail(BILUK_EARG, "batch segments must cover [0, n)");
    for (int32_t i = 0; i < nsys; ++i)
        if (seg[i + 1] < seg[i]) return fail(BILUK_EARG, "batch segments must be non-decreasing");
    return bicgstab_engine(A, M, cb, user, nsys, seg, dev_b, dev_x, dev_work, max_iters, rel_tol, stats, nullptr, 0,
                           static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// Device-driven BiCGSTAB over nsys independent systems (nsys = 1: biluk_bicgstab).
//
// Every scalar, stopping test and iteration count lives on the device: the
// epilogue kernels (FIN_B_*) run the tests of biluk_bicgstab's host loop per
// system and freeze a system once it stops (state word); when the last system
// stops, a `dead` word makes every later SpMV and preconditioner apply return
// at once.  One iteration is captured ONCE in a CUDA graph (when the
// preconditioner is a plan -- a Python callback cannot be captured) and
// replayed; the host reads the state words of iteration i-1 while iteration i
// runs, so the GPU never waits for it, and at most one replay past the stop
// is issued (all of its kernels skip).
int biluk::bicgstab_engine(biluk_op_t *A, biluk_plan_t *M, biluk_precond_fn cb, void *user, int32_t nsys,
                           const int64_t *seg, const double *dev_b, double *dev_x, void *dev_work, int64_t max_iters,
                           double rel_tol, double *stats, double *history, int64_t hist_cap, cudaStream_t stream) {
    const int64_t bs = A->o.bs;
    const int64_t len = A->o.n * bs;
    const int32_t precond = (M || cb) ? 1 : 0;
    const uint64_t vec = ((8 * uint64_t(len) + 255) / 256) * 256;
    unsigned char *w = static_cast<unsigned char *>(dev_work);
    double *r = reinterpret_cast<double *>(w + 0 * vec);
    double *rh = reinterpret_cast<double *>(w + 1 * vec);
    double *pv = reinterpret_cast<double *>(w + 2 * vec);
    double *v = reinterpret_cast<double *>(w + 3 * vec);
    double *ph = reinterpret_cast<double *>(w + 4 * vec);
    double *sv = reinterpret_cast<double *>(w + 5 * vec);
    double *sh = reinterpret_cast<double *>(w + 6 * vec);
    double *t = reinterpret_cast<double *>(w + 7 * vec);
    double *partials = reinterpret_cast<double *>(w + 8 * vec);
    double *scal = partials + int64_t(RED_BLOCKS) * MAXQ * nsys;
    int64_t *dseg = reinterpret_cast<int64_t *>(scal + int64_t(B_STRIDE) * nsys);
    int *dstate = reinterpret_cast<int *>(dseg + nsys + 1);
    int *dlive = dstate + nsys;   // alive, dead
    // the solve runs on a private non-blocking stream (capturable, unlike the
    // legacy default stream; one per host thread and device, kept), ordered
    // after / before the caller's stream
    static thread_local cudaStream_t streams[64] = {};
    static thread_local cudaEvent_t events[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(BILUK_ECUDA, "bicgstab: no device");
    if (!streams[dev] && cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess)
        return fail(BILUK_ECUDA, "bicgstab: stream setup failed");
    if (!events[dev] && cudaEventCreateWithFlags(&events[dev], cudaEventDisableTiming) != cudaSuccess)
        return fail(BILUK_ECUDA, "bicgstab: event setup failed");
    cudaStream_t gs = streams[dev];
    if (cudaEventRecord(events[dev], stream) != cudaSuccess || cudaStreamWaitEvent(gs, events[dev], 0) != cudaSuccess)
        return fail(BILUK_ECUDA, "bicgstab: stream ordering failed");
    struct Rejoin {   // the caller's stream waits for everything issued on gs
        cudaStream_t caller, gs;
        cudaEvent_t ev;
        ~Rejoin() {
            cudaEventRecord(ev, gs);
            cudaStreamWaitEvent(caller, ev, 0);
        }
    } rejoin{stream, gs, events[dev]};
    Ctx c{A, M, cb, user, gs, len, scal, partials, 0};
    c.nsys = nsys;
    c.seg = dseg;
    c.state = dstate;
    c.sstride = B_STRIDE;
    c.tol = rel_tol;
    c.alive = dlive;
    c.dead = dlive + 1;
    std::vector<int64_t> hseg(nsys + 1);
    for (int32_t i = 0; i <= nsys; ++i) hseg[i] = seg[i] * bs;
    for (int32_t i = 0; i < nsys; ++i) {
        stats[4 * i + 0] = 0; stats[4 * i + 1] = 0; stats[4 * i + 2] = INFINITY; stats[4 * i + 3] = 0;
    }
    double *dhist = nullptr;   // the residual history lives at the end of the workspace
    if (history && hist_cap > 0 && nsys == 1) {
        dhist = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(dlive + 2) + 255) & ~uintptr_t(255));
        c.hist = dhist;
        c.hcap = std::min<int64_t>(hist_cap, HIST_CAP);
    }
    const int init_live[2] = {nsys, 0};
    if (!c.err) c.err = cudaMemcpyAsync(dseg, hseg.data(), 8 * (nsys + 1), cudaMemcpyHostToDevice, c.s);
    if (!c.err) c.err = cudaMemsetAsync(dstate, 0, 4 * nsys, c.s);   // the <b, b> pass below reads it
    if (!c.err) c.err = cudaMemcpyAsync(dlive, init_live, sizeof(init_live), cudaMemcpyHostToDevice, c.s);
    if (!c.err) c.err = cudaStreamSynchronize(c.s);                   // hseg, init_live live on the host
    c.zero(dev_x);
    c.smax = 2;
    {
        Fused f{};
        f.op = 0; f.ic0 = f.ic1 = -1; f.nq = 1; f.qa[0] = dev_b; f.qb[0] = dev_b;
        c.fused(f);
        c.fin(1, S_GEN0, 0, 0, FIN_B_INIT);
    }
    c.copy(r, dev_b);
    c.copy(rh, dev_b);
    c.zero(pv);
    c.zero(v);
    const double *M_p = precond ? ph : pv;
    const double *M_s = precond ? sh : sv;
    c.skip = c.dead;
    auto iteration = [&]() -> int {
        c.smax = 0;
        Fused f{};   // p = r + beta (p - omega v)
        f.op = 2; f.u = pv; f.v = v; f.x = r; f.ic0 = S_BETA; f.ic1 = S_OMEGA; f.sgn0 = 1.0; f.nq = 0;
        c.fused(f);
        if (precond && c.apply(pv, ph) != BILUK_OK) return BILUK_ECUDA;
        c.spmv(M_p, v);
        Fused fv{};   // <r^, v> -> alpha
        fv.op = 0; fv.ic0 = fv.ic1 = -1; fv.nq = 1; fv.qa[0] = rh; fv.qb[0] = v;
        c.fused(fv);
        c.fin(1, S_RV, 0, 0, FIN_B_ALPHA);
        Fused fs{};   // s = r - alpha v ; ||s||^2 -> half-step test
        fs.op = 1; fs.u = sv; fs.x = r; fs.v = v; fs.ic0 = S_ALPHA; fs.ic1 = -1; fs.sgn0 = -1.0; fs.nq = 1;
        c.fused(fs);
        c.fin(1, S_SS, 0, 0, FIN_B_HALF);
        if (precond && c.apply(sv, sh) != BILUK_OK) return BILUK_ECUDA;
        c.spmv(M_s, t);
        Fused fd{};   // <t, t>, <t, s> -> omega
        fd.op = 0; fd.ic0 = fd.ic1 = -1; fd.nq = 2; fd.qa[0] = t; fd.qb[0] = t; fd.qa[1] = t; fd.qb[1] = sv;
        c.fused(fd);
        c.fin(2, S_TT, S_TS, 0, FIN_B_OMEGA);
        c.smax = 1;   // x += xa p^ + xw s^  (also for systems finishing at the half step)
        Fused fx{};
        fx.op = 3; fx.u = dev_x; fx.v = M_p; fx.w = M_s; fx.ic0 = S_XA; fx.ic1 = S_XW; fx.sgn0 = 1.0;
        c.fused(fx);
        c.smax = 0;   // r = s - omega t ; ||r||^2 ; rho_next = <r^, r>
        Fused fr{};
        fr.op = 1; fr.u = r; fr.x = sv; fr.v = t; fr.ic0 = S_OMEGA; fr.ic1 = -1; fr.sgn0 = -1.0; fr.nq = 2;
        fr.qa[0] = nullptr; fr.qb[0] = nullptr; fr.qa[1] = rh; fr.qb[1] = nullptr;
        c.fused(fr);
        c.fin(2, S_RR, S_RHO_NEXT, 0, FIN_B_BETA);
        return c.err ? BILUK_ECUDA : BILUK_OK;
    };
    // one iteration as a CUDA graph (plan or no preconditioner)
    cudaGraphExec_t gexec = nullptr;
    const int adopt = (!c.err && !cb && M) ? plan_adopt_stream(M, c.s) : BILUK_OK;
    if (!c.err && !cb && adopt == BILUK_OK) {
        cudaGraph_t g = nullptr;
        if (cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            const int rc = iteration();
            const cudaError_t cerr = c.err;
            const cudaError_t ec = cudaStreamEndCapture(c.s, &g);
            cudaError_t ei = cudaErrorUnknown;
            if (rc == BILUK_OK && ec == cudaSuccess && g) ei = cudaGraphInstantiate(&gexec, g, 0);
            if (ei != cudaSuccess) gexec = nullptr;
            if (std::getenv("BILUK_KRYLOV_DEBUG"))
                fprintf(stderr, "[bicgstab_engine] capture: iteration %d / %s, end %s, instantiate %s\n", rc,
                        cudaGetErrorString(cerr), cudaGetErrorString(ec), cudaGetErrorString(ei));
            if (g) cudaGraphDestroy(g);
            if (!gexec) {   // not capturable here: run the iterations eagerly
                cudaGetLastError();
                c.err = cudaSuccess;
                c.prc = BILUK_OK;
            }
        } else {
            cudaGetLastError();
        }
    }
    const bool dbg = std::getenv("BILUK_KRYLOV_DEBUG") != nullptr;   // diagnostics: graph use and loop time
    auto now = []() { return std::chrono::steady_clock::now(); };
    const auto t_cap = now();
    // host loop: replay, and look at the states of the previous iteration
    static thread_local int *hstate = nullptr;   // two pinned stop words, kept for later solves
    cudaEvent_t ev[2] = {nullptr, nullptr};
    if (!hstate && !c.err) c.err = cudaMallocHost(reinterpret_cast<void **>(&hstate), 2 * sizeof(int));
    for (cudaEvent_t &e : ev)
        if (!c.err) c.err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    int rc = BILUK_OK;
    for (int64_t it = 1; it <= max_iters && !c.err; ++it) {
        if (gexec) {
            c.err = cudaGraphLaunch(gexec, c.s);
        } else if ((rc = iteration()) != BILUK_OK) {
            break;
        }
        if (!c.err) c.err = cudaMemcpyAsync(hstate + (it & 1), c.dead, sizeof(int), cudaMemcpyDeviceToHost, c.s);
        if (!c.err) c.err = cudaEventRecord(ev[it & 1], c.s);
        if (it >= 2 && !c.err) {   // iteration it-1 is done by now, or soon: its stop word
            c.err = cudaEventSynchronize(ev[(it - 1) & 1]);
            if (!c.err && hstate[(it - 1) & 1] != 0) break;
        }
    }
    if (gexec) {
        cudaGraphExecDestroy(gexec);
        if (M && !c.err) plan_mark(M, c.s);   // later applies on other streams wait for the replays
    }
    if (!c.err) c.err = cudaStreamSynchronize(c.s);
    if (dbg)
        fprintf(stderr, "[bicgstab_engine] graph=%d loop %.3f ms\n", gexec != nullptr,
                std::chrono::duration<double, std::milli>(now() - t_cap).count());
    for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    if (c.err || rc != BILUK_OK) {
        return krylov_fail(c, nsys == 1 ? "bicgstab" : "bicgstab_batched");
    }
    // true residuals ||b_s - A_s x_s|| / ||b_s||
    c.skip = nullptr;
    c.spmv(dev_x, t);
    if (!c.err) {
        sub_kernel<<<c.sms() * 8, 256, 0, c.s>>>(t, dev_b, t, len);
        c.err = cudaGetLastError();
    }
    c.smax = 2;
    {
        Fused f{};
        f.op = 0; f.ic0 = f.ic1 = -1; f.nq = 1; f.qa[0] = t; f.qb[0] = t;
        c.fused(f);
        c.fin(1, S_GEN1, 0, 0, FIN_B_TRUE);
    }
    std::vector<double> hs(size_t(B_STRIDE) * nsys);
    if (!c.err) c.err = cudaMemcpyAsync(hs.data(), scal, 8 * hs.size(), cudaMemcpyDeviceToHost, c.s);
    if (!c.err) c.err = cudaStreamSynchronize(c.s);
    if (!c.err && dhist) {
        const int64_t nh = std::min<int64_t>(int64_t(hs[S_NH]), c.hcap);
        if (nh > 0) c.err = cudaMemcpyAsync(history, dhist, 8 * size_t(nh), cudaMemcpyDeviceToHost, c.s);
        if (!c.err) c.err = cudaStreamSynchronize(c.s);
    }
    if (c.err) return krylov_fail(c, nsys == 1 ? "bicgstab" : "bicgstab_batched");
    for (int32_t i = 0; i < nsys; ++i) {
        const double *q = hs.data() + size_t(B_STRIDE) * i;
        stats[4 * i + 0] = q[S_ITS];
        stats[4 * i + 1] = q[S_TRUE] <= rel_tol ? 1 : 0;
        stats[4 * i + 2] = q[S_TRUE];
        stats[4 * i + 3] = q[S_NH];
    }
    return M ? biluk_plan_status(M, c.s) : BILUK_OK;
}

extern "C" {

// GMRES(m), left preconditioned, MGS Arnoldi, Givens on the host (gmres.py:76-186)
int biluk_gmres(biluk_op_t *A, biluk_plan_t *M, biluk_precond_fn cb, void *user, const double *dev_b,
                double *dev_x, void *dev_work, int32_t restart, int64_t max_iters, double rel_tol, double abs_tol,
                double *stats, double *history, int64_t hist_cap, void *stream) {
    if (!A || !A->o.valued) return fail(BILUK_EARG, "operator has no values");
    if (A->o.n != A->o.ncols) return fail(BILUK_EARG, "gmres requires a square matrix");
    if (M && (!M->p.factored || M->p.n * M->p.bs != A->o.n * A->o.bs))   // vectors must match; blockings may differ
        return fail(BILUK_EARG, "preconditioner does not match the operator");
    if (restart < 1 || max_iters < 1 || !(rel_tol > 0.0) || !(abs_tol > 0.0))
        return fail(BILUK_EARG, "bad solver configuration");
    const int64_t len = A->o.n * A->o.bs;
    const int m = restart;
    const uint64_t vec = ((8 * uint64_t(len) + 255) / 256) * 256;
    unsigned char *wb = static_cast<unsigned char *>(dev_work);
    double *tmp = reinterpret_cast<double *>(wb + 0 * vec);
    double *wv = reinterpret_cast<double *>(wb + 1 * vec);
    double *z = reinterpret_cast<double *>(wb + 2 * vec);
    double *yv = reinterpret_cast<double *>(wb + 3 * vec);   // small: y coefficients
    double *V = reinterpret_cast<double *>(wb + 8 * vec);    // m+1 basis vectors
    double *partials = reinterpret_cast<double *>(wb + (8 + uint64_t(m) + 1) * vec);
    double *scal = partials + RED_BLOCKS * MAXQ;
    const int64_t ld = int64_t(vec / 8);
    Ctx c{A, M, cb, user, static_cast<cudaStream_t>(stream), len, scal, partials, 0};
    int64_t nh = 0;
    auto hist = [&](double v) {
        if (history && nh < hist_cap) history[nh] = v;
        ++nh;
    };
    auto Mop = [&](const double *in, double *out) -> int { return c.apply(in, out); };
    auto norm = [&](const double *a) -> double {
        c.dot(a, a, S_GEN0);
        double v = 0;
        c.read(&v, S_GEN0, 1);
        return std::sqrt(v);
    };
    auto true_res = [&]() -> double {   // ||b - A x||
        c.spmv(dev_x, tmp);
        if (!c.err) {
            sub_kernel<<<c.sms() * 8, 256, 0, c.s>>>(tmp, dev_b, tmp, len);
            c.err = cudaGetLastError();
        }
        return norm(tmp);
    };
    stats[0] = 0;
    stats[1] = 0;
    stats[2] = INFINITY;
    stats[3] = 0;
    c.zero(dev_x);
    const double bnorm = norm(dev_b);
    if (c.err) return krylov_fail(c, "gmres");
    if (len == 0 || bnorm == 0.0) {
        stats[1] = 1;
        stats[2] = 0;
        return BILUK_OK;
    }
    if (Mop(dev_b, z) != BILUK_OK) return krylov_fail(c, "gmres");
    double mbnorm = norm(z);
    if (mbnorm == 0.0) mbnorm = bnorm;
    double target = rel_tol;
    int64_t its = 0;
    bool breakdown = false;
    std::vector<double> H(size_t(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), col(m + 2);
    while (its < max_iters && !breakdown) {
        // z = M (b - A x)
        c.spmv(dev_x, tmp);
        if (!c.err) {
            sub_kernel<<<c.sms() * 8, 256, 0, c.s>>>(tmp, dev_b, tmp, len);
            c.err = cudaGetLastError();
        }
        if (Mop(tmp, z) != BILUK_OK) return krylov_fail(c, "gmres");
        const double beta = norm(z);
        if (c.err) return krylov_fail(c, "gmres");
        hist(beta / mbnorm);
        if (beta / mbnorm <= target || beta <= abs_tol) {
            const double tr = true_res();
            if (c.err) return krylov_fail(c, "gmres");
            if (tr / bnorm <= rel_tol) break;
            target *= 0.25;
            if (target < 1e-16) break;
            continue;
        }
        // V[0] = z / beta  (beta^2 is still in S_GEN0 from norm(z))
        if (!c.err) {
            scale_copy_kernel<<<c.sms() * 8, 256, 0, c.s>>>(V, z, len, scal, S_GEN0, 2);
            c.err = cudaGetLastError();
        }
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int used = 0;
        while (used < m && its < max_iters) {
            const int j = used;
            c.spmv(V + j * ld, tmp);
            if (Mop(tmp, wv) != BILUK_OK) return krylov_fail(c, "gmres");
            ++its;
            // MGS: h_ij = <v_i, w>; w -= h_ij v_i  (i = 0..j), then ||w||; each
            // pass fuses the previous axpy with the next dot
            c.dot(V, wv, S_H0);
            for (int i = 1; i <= j + 1; ++i) {
                Fused f{};
                f.op = 1; f.u = wv; f.x = wv; f.v = V + (i - 1) * ld; f.ic0 = S_H0 + i - 1; f.ic1 = -1; f.sgn0 = -1.0; f.nq = 1;
                if (i <= j) { f.qa[0] = V + i * ld; f.qb[0] = nullptr; }
                else { f.qa[0] = nullptr; f.qb[0] = nullptr; }
                c.fused(f);
                c.fin(1, S_H0 + i, 0, 0, FIN_NONE);
            }
            c.read(col.data(), S_H0, j + 2);
            if (c.err) return krylov_fail(c, "gmres");
            for (int i = 0; i <= j; ++i) H[size_t(i) * m + j] = col[i];
            const double hnext = std::sqrt(col[j + 1]);
            H[size_t(j + 1) * m + j] = hnext;
            for (int i = 0; i < j; ++i) {
                const double a0 = H[size_t(i) * m + j], b0 = H[size_t(i + 1) * m + j];
                H[size_t(i) * m + j] = cs[i] * a0 + sn[i] * b0;
                H[size_t(i + 1) * m + j] = -sn[i] * a0 + cs[i] * b0;
            }
            const double den = std::hypot(H[size_t(j) * m + j], H[size_t(j + 1) * m + j]);
            if (den == 0.0) {
                cs[j] = 1.0;
                sn[j] = 0.0;
            } else {
                cs[j] = H[size_t(j) * m + j] / den;
                sn[j] = H[size_t(j + 1) * m + j] / den;
            }
            H[size_t(j) * m + j] = den;
            H[size_t(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            used = j + 1;
            const double est = std::fabs(g[j + 1]) / mbnorm;
            hist(est);
            if (hnext <= abs_tol) {
                breakdown = true;
                break;
            }
            if (!c.err) {
                scale_copy_kernel<<<c.sms() * 8, 256, 0, c.s>>>(V + (j + 1) * ld, wv, len, scal, S_H0 + j + 1, 2);
                c.err = cudaGetLastError();
            }
            if (est <= target) break;
        }
        if (used) {
            for (int i = used - 1; i >= 0; --i) {
                double acc = g[i];
                for (int q = i + 1; q < used; ++q) acc -= H[size_t(i) * m + q] * y[q];
                y[i] = H[size_t(i) * m + i] != 0.0 ? acc / H[size_t(i) * m + i] : 0.0;
            }
            if (!c.err) c.err = cudaMemcpyAsync(yv, y.data(), 8 * used, cudaMemcpyHostToDevice, c.s);
            if (!c.err) {
                combo_kernel<<<c.sms() * 8, 256, 0, c.s>>>(dev_x, V, ld, len, yv, used);
                c.err = cudaGetLastError();
            }
            if (!c.err) c.err = cudaStreamSynchronize(c.s);   // y lives on the host
        }
        if (c.err) return krylov_fail(c, "gmres");
    }
    const double rel = true_res() / bnorm;
    if (c.err) return krylov_fail(c, "gmres");
    stats[0] = double(its);
    stats[1] = rel <= rel_tol ? 1 : 0;
    stats[2] = rel;
    stats[3] = double(nh);
    return M ? biluk_plan_status(M, stream) : BILUK_OK;
}

}  // extern "C"
