// extern "C" surface of libbiluk (declared in include/biluk.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "biluk_internal.h"
#include "kernels.cuh"

struct biluk_pattern {
    int64_t n = 0;
    std::vector<int32_t> rp, ci;
};

namespace biluk {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }
int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}
static int cuda_fail(cudaError_t e, const char *what) {
    return fail(BILUK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_TRY(expr, what)                          \
    do {                                              \
        cudaError_t _e = (expr);                      \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

static DevStatus *dev_status(Plan &p) { return reinterpret_cast<DevStatus *>(p.ws + p.off.status); }

// the parity-tagged sweep vectors restart at parity 0 (so the next apply, parity 1, sees no stale data)
static cudaError_t clear_tagged(Plan &p, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(p.ws + p.off.y_t, 0, 8 * plan_npos(p) * plan_vs(p), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p.ws + p.off.x_t, 0, 8 * plan_npos(p) * plan_vs(p), s);
    return e;
}

int64_t apply_bytes(const Plan &p) {
    // 8b^2(nL+nU+n) + 4(nL+nU) + 8(n+1) + 32bn
    const int64_t b = p.bs;
    return 8 * b * b * (p.nL + p.nU + p.n) + 4 * (p.nL + p.nU) + 8 * (p.n + 1) + 32 * b * p.n;
}
int64_t spmv_bytes(const Plan &p) {
    const int64_t b = p.bs;
    return 8 * b * b * p.nnzA + 4 * p.nnzA + 4 * (p.n + 1) + 16 * b * p.n;
}

}  // namespace biluk

using namespace biluk;

extern "C" {

const char *biluk_last_error(void) { return g_err.c_str(); }

int biluk_set_device(int32_t device) {
    CUDA_TRY(cudaSetDevice(device), "set device");
    return BILUK_OK;
}
const char *biluk_version(void) { return "biluk 0.1.0 (sm_100a)"; }

int biluk_symbolic(int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int32_t k, biluk_pattern_t **out,
                   int64_t *err_row) {
    if (!out) return fail(BILUK_EARG, "null output");
    *out = nullptr;
    if (k < 0) return fail(BILUK_EARG, "fill level k must be nonnegative");
    if (n < 0 || n >= INT32_MAX || (n > 0 && row_ptr[n] >= INT32_MAX))
        return fail(BILUK_EUNSUPPORTED, "pattern exceeds 2^31 entries");
    std::vector<int32_t> rp(n + 1), ci(n ? row_ptr[n] : 0);
    for (int64_t i = 0; i <= n; ++i) rp[i] = int32_t(row_ptr[i]);
    for (size_t t = 0; t < ci.size(); ++t) ci[t] = int32_t(col_idx[t]);
    auto *pat = new (std::nothrow) biluk_pattern;
    if (!pat) return fail(BILUK_ENOMEM, "out of host memory");
    pat->n = n;
    int rc = symbolic_phase(n, rp.data(), ci.data(), k, pat->rp, pat->ci, err_row);
    if (rc != BILUK_OK) {
        delete pat;
        return rc;
    }
    *out = pat;
    return BILUK_OK;
}

int64_t biluk_pattern_nnz(const biluk_pattern_t *p) { return p ? int64_t(p->ci.size()) : -1; }

int biluk_pattern_copy(const biluk_pattern_t *p, int64_t *row_ptr, int64_t *col_idx) {
    if (!p) return fail(BILUK_EARG, "null pattern");
    for (int64_t i = 0; i <= p->n; ++i) row_ptr[i] = p->rp[i];
    for (size_t t = 0; t < p->ci.size(); ++t) col_idx[t] = p->ci[t];
    return BILUK_OK;
}

void biluk_pattern_free(biluk_pattern_t *p) { delete p; }

int biluk_level_schedule(int64_t m, const int64_t *row_ptr, const int64_t *col_idx, int32_t upper,
                         int64_t *level_of_row, int64_t *num_levels) {
    if (m < 0) return fail(BILUK_EARG, "negative dimension");
    for (int64_t i = 0; i < m; ++i)
        for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
            const int64_t j = col_idx[t];
            if (j < 0 || j >= m || (upper ? j <= i : j >= i))
                return fail(BILUK_ESTRUCT, std::string("entry on or across the diagonal in a ") +
                                               (upper ? "upper" : "lower") + " operand");
        }
    level_schedule(m, row_ptr, col_idx, upper != 0, level_of_row, num_levels);
    return BILUK_OK;
}

int biluk_plan_create(int32_t bs, int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int32_t k,
                      biluk_plan_t **out, int64_t *err_row) {
    return biluk_plan_create_ex(bs, n, row_ptr, col_idx, k, 0, out, err_row);
}

int biluk_plan_create_ex(int32_t bs, int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int32_t k,
                         int32_t flags, biluk_plan_t **out, int64_t *err_row) {
    if (!out) return fail(BILUK_EARG, "null output");
    *out = nullptr;
    auto *h = new (std::nothrow) biluk_plan;
    if (!h) return fail(BILUK_ENOMEM, "out of host memory");
    int rc = plan_analyse(h->p, bs, n, row_ptr, col_idx, k, err_row);
    if (rc != BILUK_OK) {
        delete h;
        return rc;
    }
    if (flags & BILUK_PLAN_FACTOR_ONLY) {   // materialize + factorize only: no sweep plan, no apply
        int dev0 = 0, sms0 = 148, smem0 = 227 * 1024;
        if (cudaGetDevice(&dev0) == cudaSuccess) {
            cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0);
            cudaDeviceGetAttribute(&smem0, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev0);
        } else {
            cudaGetLastError();
        }
        h->p.engine = 0;
        h->p.factor_only = true;
        plan_layout(h->p, sms0, size_t(smem0));
        *out = h;
        return BILUK_OK;
    }
    int dev = 0, sms = 148, smem = 227 * 1024;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    } else {
        cudaGetLastError();   // no device here: plan for a B200
    }
    // apply engine, from B200 measurements (tools/engine_compare.py, DESIGN.md
    // §3): the partitioned sweep wins while its records per part stay few --
    // always for ILU(0) with b <= 3 (grid columns); ILU(0) with b = 4 up to
    // ~400 records per part (100^3 yes, 128^3 no); with fill (contiguous
    // parts) up to ~1500 (128^3 ILU(2): 1352, yes).  Larger blocks and
    // batches of many systems go to the tiled level-order sweep.
    // BILUK_ENGINE overrides.
    Plan &P = h->p;
    const char *env = std::getenv("BILUK_ENGINE");
    // (very large operators -- e.g. the 64-system batch, 16.8 M block rows --
    // plan far over the records-per-part limit; they skip the partitioned
    // planning, which would only be discarded, outright)
    P.engine = (bs <= 4 && n <= (int64_t(1) << 22)) ? 1 : 0;
    if (env) P.engine = std::atoi(env) == 0 ? 0 : 1;
    // ILU(0) of a 7-point block grid: the grid sweep (engine 2) when it plans
    const bool want_grid = env ? std::atoi(env) == 2 : false;
    if (want_grid) {
        rc = plan_gsweep(P, sms, size_t(smem));
        if (rc == BILUK_OK) {
            P.engine = 2;
        } else {
            P.gs = GSweep{};
        }
    }
    if (P.engine == 1) {
        const auto t_ps = std::chrono::steady_clock::now();
        rc = plan_psweep(P, sms, size_t(smem), 0);
        if (std::getenv("BILUK_PLAN_TIMING"))
            std::fprintf(stderr, "[plan] partitioned sweep records %.3f s\n",
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t_ps).count());
        const double per_part = P.ps.P > 0 ? double(P.ps.rec.size()) / P.ps.P : 0.0;
        const double limit = k >= 1 ? 1500.0 : (bs <= 3 ? 1e30 : 400.0);
        // three compute groups (blocks read at the products) measured faster
        // than two (blocks staged in registers) for every case; BILUK_GROUPS=2
        // selects the two-group kernel
        P.ps.groups = 3;
        // producer warps (each streams its share of the records into its share
        // of the ring): four with fill -- smaller records, more copies in
        // flight (128^3 ILU(2) 3081 vs 3162 us with one, 3478 with two; 100^3 b4
        // ILU(1) 1609 vs 1686; 128^3 ILU(1) 1478 vs 1511; 64^3 622 vs 626);
        // two for ILU(0), whose large U' records need the bigger shares (511 vs
        // 526 us with four, 668 with one)
        P.ps.nprod = (k >= 1 && bs <= 4) ? 4 : 2;
        if (const char *g = std::getenv("BILUK_NPROD")) {
            const int v = std::atoi(g);
            P.ps.nprod = (v >= 3 && v <= 4 && bs <= 4) ? v : (v == 1 ? 1 : 2);
        }
        if (const char *g = std::getenv("BILUK_GROUPS")) P.ps.groups = std::atoi(g) == 3 ? 3 : 2;
        if (rc == BILUK_EUNSUPPORTED || (rc == BILUK_OK && !env && per_part > limit)) {
            P.engine = 0;
            P.ps = PSweep{};
        } else if (rc != BILUK_OK) {
            delete h;
            return rc;
        }
    }
    if (P.engine == 0) {
        rc = plan_tiles(P);
        // a tile stages all its rows padded to its longest row: one stage must
        // fit in shared memory (very long rows -- e.g. an arrowhead -- do not)
        const int64_t stage = std::max<int64_t>(128, std::max(P.sl.max_rec, P.su.max_rec));
        if (rc == BILUK_OK && stage + 16 > int64_t(smem) - 4096)
            rc = fail(BILUK_EUNSUPPORTED, "a factor row has " + std::to_string(std::max(P.sl.max_slots, P.su.max_slots)) +
                                              " off-diagonal blocks: its sweep tile (" + std::to_string(stage) +
                                              " bytes) exceeds shared memory");
        if (rc != BILUK_OK) {
            delete h;
            return rc;
        }
    }
    plan_layout(P, sms, size_t(smem));
    *out = h;
    return BILUK_OK;
}

void biluk_plan_destroy(biluk_plan_t *plan) { delete plan; }

uint64_t biluk_plan_workspace_bytes(const biluk_plan_t *plan) { return plan ? plan->p.off.total : 0; }

int biluk_plan_bind(biluk_plan_t *plan, void *dev_workspace, uint64_t bytes, void *stream) {
    if (!plan) return fail(BILUK_EARG, "null plan");
    Plan &p = plan->p;
    if (bytes < p.off.total) return fail(BILUK_EARG, "workspace too small");
    if (reinterpret_cast<uintptr_t>(dev_workspace) % 256) return fail(BILUK_EARG, "workspace must be 256-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    p.ws = static_cast<unsigned char *>(dev_workspace);
    // launch configuration check: the persistent sweep needs every CTA resident
    int per_sm = 1;
    if (p.factor_only) {
    } else if (p.engine == 2) {
        CUDA_TRY(gsweep_occupancy(p, &per_sm), "sweep occupancy");
    } else if (p.engine == 1) {
        CUDA_TRY(psweep_occupancy(p, &per_sm), "sweep occupancy");
    } else {
        CUDA_TRY(sweep_occupancy(p, &per_sm), "sweep occupancy");
    }
    if (per_sm < 1) return fail(BILUK_EUNSUPPORTED, "sweep kernel does not fit on an SM");
    auto up = [&](uint64_t off, const void *src, size_t n) -> cudaError_t {
        if (n == 0) return cudaSuccess;
        return cudaMemcpyAsync(p.ws + off, src, n, cudaMemcpyHostToDevice, s);
    };
    CUDA_TRY(up(p.off.p_rp, p.p_rp.data(), 4 * p.p_rp.size()), "upload");
    CUDA_TRY(up(p.off.p_ci, p.p_ci.data(), 4 * p.p_ci.size()), "upload");
    CUDA_TRY(up(p.off.p_diag, p.p_diag.data(), 4 * p.p_diag.size()), "upload");
    CUDA_TRY(up(p.off.a2p, p.a2p.data(), 4 * p.a2p.size()), "upload");
    CUDA_TRY(up(p.off.forder, p.forder.data(), 4 * p.forder.size()), "upload");
    CUDA_TRY(up(p.off.sl_rows, p.sl.tile_rows.data(), 4 * p.sl.tile_rows.size()), "upload");
    CUDA_TRY(up(p.off.sl_meta, p.sl.meta.data(), sizeof(TileMeta) * p.sl.meta.size()), "upload");
    CUDA_TRY(up(p.off.su_rows, p.su.tile_rows.data(), 4 * p.su.tile_rows.size()), "upload");
    CUDA_TRY(up(p.off.su_meta, p.su.meta.data(), sizeof(TileMeta) * p.su.meta.size()), "upload");
    CUDA_TRY(up(p.off.lvl_tiles, p.lvl_tiles.data(), 4 * p.lvl_tiles.size()), "upload");
    CUDA_TRY(cudaMemsetAsync(p.ws + p.off.lvl_cnt, 0, 4 * p.lvl_tiles.size(), s), "memset");
    CUDA_TRY(up(p.off.ps_info, p.ps.rec.data(), sizeof(PRecInfo) * p.ps.rec.size()), "upload");
    CUDA_TRY(up(p.off.ps_part, p.ps.part_rec.data(), 4 * p.ps.part_rec.size()), "upload");
    CUDA_TRY(up(p.off.ps_idx, p.ps.idx.data(), 4 * p.ps.idx.size()), "upload");
    CUDA_TRY(up(p.off.ps_vmap, p.ps.vmap.data(), 4 * p.ps.vmap.size()), "upload");
    if (p.engine == 1) {   // position -> row (the b permutation gathers)
        std::vector<int32_t> lrow(p.ps.posL.size());
        for (size_t i = 0; i < lrow.size(); ++i) lrow[size_t(p.ps.posL[i])] = int32_t(i);
        CUDA_TRY(cudaMemcpyAsync(p.ws + p.off.ps_posl, lrow.data(), 4 * lrow.size(), cudaMemcpyHostToDevice, s),
                 "upload");
        CUDA_TRY(cudaStreamSynchronize(s), "upload sync");
    }
    if (p.engine == 2) {
        CUDA_TRY(up(p.off.gs_part, p.gs.part.data(), sizeof(GPart) * p.gs.part.size()), "upload");
        CUDA_TRY(up(p.off.gs_rec, p.gs.rec.data(), sizeof(GRec) * p.gs.rec.size()), "upload");
        CUDA_TRY(up(p.off.gs_lo, p.gs.rec_lo.data(), 4 * p.gs.rec_lo.size()), "upload");
        CUDA_TRY(up(p.off.gs_cols, p.gs.cols.data(), 4 * p.gs.cols.size()), "upload");
    }
    CUDA_TRY(up(p.off.pos_l, p.sl.pos.data(), 4 * p.sl.pos.size()), "upload");
    CUDA_TRY(up(p.off.pos_u, p.su.pos.data(), 4 * p.su.pos.size()), "upload");
    // parity-tagged vectors start at parity 0 everywhere; the first apply uses parity 1
    CUDA_TRY(clear_tagged(p, s), "memset");
    DevStatus init{};
    init.epoch = 1;
    init.ferr_row = (long long)INT64_MAX;
    CUDA_TRY(cudaMemcpyAsync(p.ws + p.off.status, &init, sizeof(init), cudaMemcpyHostToDevice, s), "upload");
    CUDA_TRY(cudaStreamSynchronize(s), "bind sync");
    p.bound = true;
    p.factored = false;
    return BILUK_OK;
}

static int split_and_pack(Plan &p, cudaStream_t s);

int biluk_plan_factor(biluk_plan_t *plan, const double *dev_a_vals, void *stream, int64_t *err_row) {
    if (!plan || !plan->p.bound) return fail(BILUK_EARG, "plan is not bound to a workspace");
    Plan &p = plan->p;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevStatus *st = dev_status(p);
    {
        int32_t z[2] = {0, 0};
        long long big = (long long)INT64_MAX;
        CUDA_TRY(cudaMemcpyAsync(&st->status, z, sizeof(z), cudaMemcpyHostToDevice, s), "status reset");
        CUDA_TRY(cudaMemcpyAsync(&st->ferr_row, &big, sizeof(big), cudaMemcpyHostToDevice, s), "status reset");
    }
    CUDA_TRY(launch_materialize(p, dev_a_vals, s), "materialize");
    CUDA_TRY(launch_factor(p, s), "factorize");
    DevStatus h{};
    CUDA_TRY(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s), "status read");
    CUDA_TRY(cudaStreamSynchronize(s), "factorize sync");
    if (h.fstatus != 0) {
        p.factored = false;
        if (err_row) *err_row = h.ferr_row;
        if (h.fstatus == BILUK_EZEROPIVOT)
            return fail(BILUK_EZEROPIVOT, "zero pivot at row " + std::to_string(h.ferr_row));
        return fail(BILUK_ESINGULAR, "singular diagonal block at row " + std::to_string(h.ferr_row));
    }
    if (p.factor_only) return fail(BILUK_EARG, "plan was created for factorization only (biluk_plan_factor_lu)");
    return split_and_pack(p, s);
}

static int split_and_pack(Plan &p, cudaStream_t s) {
    CUDA_TRY(launch_split(p, s), "split");
    if (p.engine == 2) {
        CUDA_TRY(launch_gpack(p, s), "pack");
    } else if (p.engine == 1) {
        CUDA_TRY(launch_ppack(p, s), "pack");
    } else {
        CUDA_TRY(launch_pack(p, s), "pack");
    }
    CUDA_TRY(cudaStreamSynchronize(s), "pack sync");
    p.factored = true;
    return BILUK_OK;
}

static void reset_fstatus(Plan &p, cudaStream_t s) {
    DevStatus *st = dev_status(p);
    int32_t z[2] = {0, 0};
    long long big = (long long)INT64_MAX;
    cudaMemcpyAsync(&st->status, z, sizeof(z), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(&st->ferr_row, &big, sizeof(big), cudaMemcpyHostToDevice, s);
}

static int read_fstatus(Plan &p, cudaStream_t s, int64_t *err_row) {
    DevStatus h{};
    CUDA_TRY(cudaMemcpyAsync(&h, dev_status(p), sizeof(h), cudaMemcpyDeviceToHost, s), "status read");
    CUDA_TRY(cudaStreamSynchronize(s), "factorize sync");
    if (h.fstatus != 0) {
        if (err_row) *err_row = h.ferr_row;
        if (h.fstatus == BILUK_EZEROPIVOT) return fail(BILUK_EZEROPIVOT, "zero pivot at row " + std::to_string(h.ferr_row));
        return fail(BILUK_ESINGULAR, "singular diagonal block at row " + std::to_string(h.ferr_row));
    }
    return BILUK_OK;
}

int biluk_plan_factor_lu(biluk_plan_t *plan, const double *dev_a_vals, double *dev_out_vals, void *stream,
                         int64_t *err_row) {
    if (!plan || !plan->p.bound) return fail(BILUK_EARG, "plan is not bound to a workspace");
    Plan &p = plan->p;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    reset_fstatus(p, s);
    CUDA_TRY(launch_materialize(p, dev_a_vals, s), "materialize");
    CUDA_TRY(launch_factor(p, s), "factorize");
    const int rc = read_fstatus(p, s, err_row);
    if (rc != BILUK_OK) return rc;
    const size_t bytes = size_t(p.nnzP) * p.bs * p.bs * 8;
    if (bytes) CUDA_TRY(cudaMemcpyAsync(dev_out_vals, p.ws + p.off.pvals, bytes, cudaMemcpyDeviceToDevice, s), "copy");
    CUDA_TRY(cudaStreamSynchronize(s), "factorize sync");
    p.factored = false;
    return BILUK_OK;
}

int biluk_plan_load_factored(biluk_plan_t *plan, const double *dev_lu_vals, void *stream, int64_t *err_row) {
    if (!plan || !plan->p.bound) return fail(BILUK_EARG, "plan is not bound to a workspace");
    Plan &p = plan->p;
    if (p.factor_only) return fail(BILUK_EARG, "plan was created for factorization only");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    reset_fstatus(p, s);
    const size_t bytes = size_t(p.nnzP) * p.bs * p.bs * 8;
    if (bytes) CUDA_TRY(cudaMemcpyAsync(p.ws + p.off.pvals, dev_lu_vals, bytes, cudaMemcpyDeviceToDevice, s), "load");
    CUDA_TRY(launch_diag_invert(p, s), "split");
    const int rc = read_fstatus(p, s, err_row);
    if (rc != BILUK_OK) {
        p.factored = false;
        return rc;
    }
    return split_and_pack(p, s);
}

static int apply_launch(biluk_plan_t *plan, const double *dev_b, double *dev_x, cudaStream_t stream,
                        const int *skip);

int biluk_plan_apply(biluk_plan_t *plan, const double *dev_b, double *dev_x, void *stream) {
    return biluk::plan_apply(plan, dev_b, dev_x, static_cast<cudaStream_t>(stream), nullptr);
}

}  // extern "C"

// the apply with an optional device skip word (*skip != 0: every kernel of the
// apply returns at once -- Krylov iterations captured in a CUDA graph after
// the solve stopped)
int biluk::plan_apply(biluk_plan_t *plan, const double *dev_b, double *dev_x, cudaStream_t st, const int *skip) {
    if (!plan || !plan->p.factored) return fail(BILUK_EARG, "plan is not factored");
    if (plan->p.factor_only) return fail(BILUK_EARG, "plan was created for factorization only");
    Plan &p = plan->p;
    if (p.n == 0) return BILUK_OK;
    if (dev_b == dev_x) return fail(BILUK_EARG, "output may not alias the right-hand side");
    // applies of one plan share its workspace (tagged vectors, epoch): order an
    // apply on a new stream after the previous one.  Inside a stream capture
    // the graph orders them; the capturing code re-marks the plan afterwards
    // (plan_mark), since an event recorded in a capture cannot be waited on
    // outside it.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(st, &cap), "apply");
    const bool capturing = cap != cudaStreamCaptureStatusNone;
    if (!capturing && plan->last_ev && plan->last_stream != st)
        CUDA_TRY(cudaStreamWaitEvent(st, plan->last_ev, 0), "apply");
    int rc = apply_launch(plan, dev_b, dev_x, st, skip);
    if (rc != BILUK_OK) return rc;
    if (capturing) return BILUK_OK;
    return plan_mark(plan, st);
}

// the plan's last apply was issued on `st` (outside any capture)
int biluk::plan_mark(biluk_plan_t *plan, cudaStream_t st) {
    if (!plan->last_ev) CUDA_TRY(cudaEventCreateWithFlags(&plan->last_ev, cudaEventDisableTiming), "apply");
    CUDA_TRY(cudaEventRecord(plan->last_ev, st), "apply");
    plan->last_stream = st;
    return BILUK_OK;
}

// make `st` the stream of the plan's next apply without capturing a wait:
// called before a CUDA graph capture on st
int biluk::plan_adopt_stream(biluk_plan_t *plan, cudaStream_t st) {
    if (plan->last_ev && plan->last_stream != st) CUDA_TRY(cudaStreamWaitEvent(st, plan->last_ev, 0), "apply");
    plan->last_stream = st;
    return BILUK_OK;
}

extern "C" {

static int apply_launch(biluk_plan_t *plan, const double *dev_b, double *dev_x, cudaStream_t stream,
                        const int *skip) {
    Plan &p = plan->p;
    if (p.engine == 2) {
        GSweepArgs a{};
        a.parts = reinterpret_cast<const GPart *>(p.ws + p.off.gs_part);
        a.recs = reinterpret_cast<const GRec *>(p.ws + p.off.gs_rec);
        a.cols = reinterpret_cast<const int32_t *>(p.ws + p.off.gs_cols);
        a.stream = p.ws + p.off.gs_stream;
        a.b = dev_b;
        a.y = reinterpret_cast<double *>(p.ws + p.off.gs_y);
        a.out = dev_x;
        a.y_t = reinterpret_cast<double *>(p.ws + p.off.y_t);
        a.x_t = reinterpret_cast<double *>(p.ws + p.off.x_t);
        a.st = dev_status(p);
        a.skip_flag = skip;
        a.timeout_ns = 2000000000ull;
        a.nx = p.gs.nx;
        a.ny = p.gs.ny;
        a.nz = p.gs.nz;
        a.slot_bytes = p.gs.slot_bytes;
        a.kslots = p.gs.kslots;
        a.trace = p.trace;
        a.nrec_total = int64_t(p.gs.rec.size());
        if (plan->tev[0]) CUDA_TRY(cudaEventRecord(plan->tev[0], static_cast<cudaStream_t>(stream)), "apply");
        CUDA_TRY(launch_gsweep(p, a, static_cast<cudaStream_t>(stream)), "apply");
        if (plan->tev[1]) CUDA_TRY(cudaEventRecord(plan->tev[1], static_cast<cudaStream_t>(stream)), "apply");
        return BILUK_OK;
    }
    if (p.engine == 1) {
        PSweepArgs a{};
        a.rec = reinterpret_cast<const PRecInfo *>(p.ws + p.off.ps_info);
        a.recs = p.ws + p.off.ps_rec;
        a.part_rec = reinterpret_cast<const int32_t *>(p.ws + p.off.ps_part);
        a.b = dev_b;
        a.y_t = reinterpret_cast<double *>(p.ws + p.off.y_t);
        a.x_t = reinterpret_cast<double *>(p.ws + p.off.x_t);
        a.out = dev_x;
        a.st = dev_status(p);
        a.skip_flag = skip;
        a.timeout_ns = 2000000000ull;
        a.ring_mask = p.ps.ring - 1;
        a.data_bytes = uint32_t(p.ps.data_ring);
        a.trace = p.trace;
        a.nrec_total = int64_t(p.ps.rec.size());
        a.b_perm = reinterpret_cast<double *>(p.ws + p.off.ps_bperm);
        a.y_u = reinterpret_cast<double *>(p.ws + p.off.ps_yu);
        CUDA_TRY(launch_permute_b(p, dev_b, static_cast<cudaStream_t>(stream), skip), "apply");
        if (plan->tev[0]) CUDA_TRY(cudaEventRecord(plan->tev[0], static_cast<cudaStream_t>(stream)), "apply");
        CUDA_TRY(launch_psweep(p, a, static_cast<cudaStream_t>(stream)), "apply");
        if (plan->tev[1]) CUDA_TRY(cudaEventRecord(plan->tev[1], static_cast<cudaStream_t>(stream)), "apply");
        return BILUK_OK;
    }
    SweepArgs a{};
    a.meta_l = reinterpret_cast<const TileMeta *>(p.ws + p.off.sl_meta);
    a.meta_u = reinterpret_cast<const TileMeta *>(p.ws + p.off.su_meta);
    a.rec_l = p.ws + p.off.sl_rec;
    a.rec_u = p.ws + p.off.su_rec;
    a.nl = p.sl.ntiles;
    a.nu = p.su.ntiles;
    a.b = dev_b;
    a.y_t = reinterpret_cast<double *>(p.ws + p.off.y_t);
    a.x_t = reinterpret_cast<double *>(p.ws + p.off.x_t);
    a.npos = plan_npos(p);
    a.out = dev_x;
    a.st = dev_status(p);
    a.skip_flag = skip;
    a.stages = p.sweep_stages;
    a.stage_bytes = int(p.stage_bytes);
    a.timeout_ns = 2000000000ull;
    a.lvl_tiles = reinterpret_cast<const uint32_t *>(p.ws + p.off.lvl_tiles);
    a.lvl_cnt = reinterpret_cast<uint32_t *>(p.ws + p.off.lvl_cnt);
    a.nlev_l = p.nlev_L;
    a.nlev_total = p.nlev_L + p.nlev_U;
    a.gap = p.tune.gap;
    a.coarse_sleep_ns = p.tune.coarse_sleep_ns;
    a.fine_sleep_ns = p.tune.fine_sleep_ns;
    a.poll_all = p.tune.poll_all;
    a.probe = p.tune.probe;
    a.probe_sleep_ns = p.tune.probe_sleep_ns;
    a.trace = p.trace;
    a.trace_mode = p.tune.trace_mode;
    if (plan->tev[0]) CUDA_TRY(cudaEventRecord(plan->tev[0], static_cast<cudaStream_t>(stream)), "apply");
    CUDA_TRY(launch_sweep(p, a, static_cast<cudaStream_t>(stream)), "apply");
    if (plan->tev[1]) CUDA_TRY(cudaEventRecord(plan->tev[1], static_cast<cudaStream_t>(stream)), "apply");
    return BILUK_OK;
}

int biluk_plan_set_timing(biluk_plan_t *plan, int32_t on) {
    if (!plan) return fail(BILUK_EARG, "null plan");
    for (cudaEvent_t &e : plan->tev) {
        if (on && !e) CUDA_TRY(cudaEventCreate(&e), "set_timing");
        if (!on && e) {
            cudaEventDestroy(e);
            e = nullptr;
        }
    }
    return BILUK_OK;
}

int biluk_plan_sweep_ms(biluk_plan_t *plan, float *ms) {
    if (!plan || !ms) return fail(BILUK_EARG, "null argument");
    if (!plan->tev[0]) return fail(BILUK_EARG, "timing is off (biluk_plan_set_timing)");
    CUDA_TRY(cudaEventSynchronize(plan->tev[1]), "sweep_ms");
    CUDA_TRY(cudaEventElapsedTime(ms, plan->tev[0], plan->tev[1]), "sweep_ms");
    return BILUK_OK;
}

int biluk_plan_records(const biluk_plan_t *plan, void *out, int64_t max_records) {
    if (!plan) return fail(BILUK_EARG, "null plan");
    const PSweep &ps = plan->p.ps;
    const int64_t n = std::min<int64_t>(max_records, int64_t(ps.rec.size()));
    if (out && n > 0) std::memcpy(out, ps.rec.data(), size_t(n) * sizeof(PRecInfo));
    return int(std::min<int64_t>(int64_t(ps.rec.size()), INT32_MAX));
}

int biluk_plan_tile_levels(const biluk_plan_t *plan, int32_t *levels) {
    if (!plan) return fail(BILUK_EARG, "null plan");
    const Plan &p = plan->p;
    int64_t q = 0;
    for (const TileMeta &m : p.sl.meta) levels[q++] = m.level;
    for (const TileMeta &m : p.su.meta) levels[q++] = p.nlev_L + m.level;
    return BILUK_OK;
}

int biluk_plan_set_trace(biluk_plan_t *plan, void *dev_trace) {
    if (!plan) return fail(BILUK_EARG, "null plan");
    plan->p.trace = static_cast<unsigned long long *>(dev_trace);
    return BILUK_OK;
}

int biluk_plan_tune(biluk_plan_t *plan, const char *key, int64_t value) {
    if (!plan || !key) return fail(BILUK_EARG, "null argument");
    SweepTune &t = plan->p.tune;
    const std::string k(key);
    if (k == "gap") t.gap = int(value);
    else if (k == "coarse_sleep_ns") t.coarse_sleep_ns = int(value);
    else if (k == "fine_sleep_ns") t.fine_sleep_ns = int(value);
    else if (k == "warps") t.warps = int(value);
    else if (k == "poll_all") t.poll_all = int(value);
    else if (k == "probe") t.probe = int(value);
    else if (k == "probe_sleep_ns") t.probe_sleep_ns = int(value);
    else if (k == "trace_mode") t.trace_mode = int(value);
    else return fail(BILUK_EARG, "unknown tuning key " + k);
    return BILUK_OK;
}

int biluk_plan_status(biluk_plan_t *plan, void *stream) {
    if (!plan || !plan->p.bound) return fail(BILUK_EARG, "plan is not bound");
    Plan &p = plan->p;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t code = 0;
    CUDA_TRY(cudaMemcpyAsync(&code, &dev_status(p)->status, 4, cudaMemcpyDeviceToHost, s), "status read");
    CUDA_TRY(cudaStreamSynchronize(s), "status sync");
    if (code != 0) {
        // the tagged vectors are in an unknown state: restart the parity protocol
        int32_t z = 0;
        uint32_t one = 1, zero = 0;
        CUDA_TRY(cudaMemcpyAsync(&dev_status(p)->status, &z, 4, cudaMemcpyHostToDevice, s), "status reset");
        CUDA_TRY(cudaMemcpyAsync(&dev_status(p)->epoch, &one, 4, cudaMemcpyHostToDevice, s), "status reset");
        CUDA_TRY(cudaMemcpyAsync(&dev_status(p)->done_ctas, &zero, 4, cudaMemcpyHostToDevice, s), "status reset");
        CUDA_TRY(cudaMemcpyAsync(&dev_status(p)->prefix, &zero, 4, cudaMemcpyHostToDevice, s), "status reset");
        CUDA_TRY(cudaMemsetAsync(p.ws + p.off.lvl_cnt, 0, 4 * p.lvl_tiles.size(), s), "memset");
        CUDA_TRY(clear_tagged(p, s), "memset");
        CUDA_TRY(cudaStreamSynchronize(s), "status sync");
        return fail(code, "device dependency wait timed out in the triangular sweep");
    }
    return BILUK_OK;
}

int biluk_plan_info(const biluk_plan_t *plan, int64_t *info, int32_t ninfo) {
    if (!plan) return fail(BILUK_EARG, "null plan");
    const Plan &p = plan->p;
    const bool g2 = p.engine == 2;
    const int64_t v[] = {p.n,          p.bs,         p.k,           p.nnzA,          p.nnzP,
                         p.nL,         p.nU,         p.nlev_L,      p.nlev_U,        p.sl.ntiles,
                         p.su.ntiles,  rows_per_tile(p.bs), int64_t(p.off.total), apply_bytes(p), spmv_bytes(p),
                         p.sweep_ctas, p.sweep_warps, p.sweep_stages, p.stage_bytes,
                         std::max(p.sl.max_slots, p.su.max_slots), p.engine, g2 ? p.gs.P : p.ps.P,
                         g2 ? int64_t(p.gs.rec.size()) : int64_t(p.ps.rec.size()), int64_t(p.ps.est_us * 1000.0),
                         g2 ? p.gs.stream_bytes : p.ps.rec_total, p.ps.nglob_total, g2 ? 1 : p.ps.partition,
                         g2 ? p.gs.py : p.ps.split[0], g2 ? p.gs.pz : p.ps.split[1]};
    const int nv = int(sizeof(v) / sizeof(v[0]));
    for (int i = 0; i < ninfo; ++i) info[i] = i < nv ? v[i] : 0;
    return BILUK_OK;
}

int biluk_plan_copy_factors(biluk_plan_t *plan, int64_t *L_row_ptr, int64_t *L_col_idx, double *L_vals, double *dinv,
                            int64_t *U_row_ptr, int64_t *U_col_idx, double *U_vals, void *stream) {
    if (!plan || !plan->p.factored) return fail(BILUK_EARG, "plan is not factored");
    Plan &p = plan->p;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t bs2 = int64_t(p.bs) * p.bs;
    std::vector<double> pv(size_t(p.nnzP * bs2)), dv(size_t(p.n * bs2));
    CUDA_TRY(cudaMemcpyAsync(pv.data(), p.ws + p.off.pvals, 8 * pv.size(), cudaMemcpyDeviceToHost, s), "copy");
    CUDA_TRY(cudaMemcpyAsync(dv.data(), p.ws + p.off.dinv, 8 * dv.size(), cudaMemcpyDeviceToHost, s), "copy");
    CUDA_TRY(cudaStreamSynchronize(s), "copy sync");
    int64_t lq = 0, uq = 0;
    if (L_row_ptr) L_row_ptr[0] = 0;
    if (U_row_ptr) U_row_ptr[0] = 0;
    for (int64_t i = 0; i < p.n; ++i) {
        for (int32_t t = p.p_rp[i]; t < p.p_rp[i + 1]; ++t) {
            if (t < p.p_diag[i]) {
                if (L_col_idx) L_col_idx[lq] = p.p_ci[t];
                if (L_vals) std::memcpy(L_vals + lq * bs2, pv.data() + int64_t(t) * bs2, 8 * bs2);
                ++lq;
            } else if (t > p.p_diag[i]) {
                if (U_col_idx) U_col_idx[uq] = p.p_ci[t];
                if (U_vals) std::memcpy(U_vals + uq * bs2, pv.data() + int64_t(t) * bs2, 8 * bs2);
                ++uq;
            }
        }
        if (L_row_ptr) L_row_ptr[i + 1] = lq;
        if (U_row_ptr) U_row_ptr[i + 1] = uq;
        if (dinv)   // column-major on the device -> row-major (n, bs, bs)
            for (int r = 0; r < p.bs; ++r)
                for (int c = 0; c < p.bs; ++c) dinv[i * bs2 + r * p.bs + c] = dv[i * bs2 + c * p.bs + r];
    }
    return BILUK_OK;
}

int biluk_op_create(int32_t bs, int64_t n_block_rows, int64_t n_block_cols, const int64_t *row_ptr,
                    const int64_t *col_idx, biluk_op_t **out) {
    if (!out) return fail(BILUK_EARG, "null output");
    *out = nullptr;
    auto *h = new (std::nothrow) biluk_op;
    if (!h) return fail(BILUK_ENOMEM, "out of host memory");
    int rc = op_analyse(h->o, bs, n_block_rows, n_block_cols, row_ptr, col_idx);
    if (rc != BILUK_OK) {
        delete h;
        return rc;
    }
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    else
        cudaGetLastError();
    h->o.num_sms = sms;
    *out = h;
    return BILUK_OK;
}

void biluk_op_destroy(biluk_op_t *op) { delete op; }

uint64_t biluk_op_workspace_bytes(const biluk_op_t *op) { return op ? op->o.off.total : 0; }

int biluk_op_bind(biluk_op_t *op, void *dev_workspace, uint64_t bytes, void *stream) {
    if (!op) return fail(BILUK_EARG, "null operator");
    Op &o = op->o;
    if (bytes < o.off.total) return fail(BILUK_EARG, "workspace too small");
    if (reinterpret_cast<uintptr_t>(dev_workspace) % 256) return fail(BILUK_EARG, "workspace must be 256-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    o.ws = static_cast<unsigned char *>(dev_workspace);
    if (o.rp.size()) CUDA_TRY(cudaMemcpyAsync(o.ws + o.off.rp, o.rp.data(), 4 * o.rp.size(), cudaMemcpyHostToDevice, s), "upload");
    if (o.ci.size()) CUDA_TRY(cudaMemcpyAsync(o.ws + o.off.ci, o.ci.data(), 4 * o.ci.size(), cudaMemcpyHostToDevice, s), "upload");
    if (o.meta.size())
        CUDA_TRY(cudaMemcpyAsync(o.ws + o.off.meta, o.meta.data(), sizeof(TileMeta) * o.meta.size(),
                                 cudaMemcpyHostToDevice, s),
                 "upload");
    CUDA_TRY(cudaStreamSynchronize(s), "bind sync");
    o.bound = true;
    o.valued = false;
    return BILUK_OK;
}

int biluk_op_set_values(biluk_op_t *op, const double *dev_vals, void *stream) {
    if (!op || !op->o.bound) return fail(BILUK_EARG, "operator is not bound to a workspace");
    CUDA_TRY(launch_pack_ell(op->o, dev_vals, static_cast<cudaStream_t>(stream)), "pack");
    op->o.valued = true;
    return BILUK_OK;
}

int biluk_op_spmv(biluk_op_t *op, const double *dev_x, double *dev_y, void *stream) {
    if (!op || !op->o.valued) return fail(BILUK_EARG, "operator has no values");
    if (op->o.n == 0) return BILUK_OK;
    CUDA_TRY(launch_spmv(op->o, dev_x, dev_y, nullptr, static_cast<cudaStream_t>(stream)), "spmv");
    return BILUK_OK;
}

}  // extern "C"
