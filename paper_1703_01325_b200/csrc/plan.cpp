// Host-side analysis of the block pattern: the ILU(k) symbolic phase, the
// block level sets of both triangles and the level-ordered tile layout that
// the device sweeps stream.  Integer work only; everything here is exact.
//
// Reference stages replaced (paths relative to /root/reference/pkg/src/blockiluk):
//   extract_point_pattern  sparse.py:261-275   (we read row_ptr/col_idx directly)
//   symbolic_phase         symbolic.py:27-72
//   materialize (indices)  factor.py:83-121    (A slot -> P' slot map)
//   build_level_schedule   trisolve.py:98-118  (block granularity for execution)
#include <algorithm>
#include <string>
#include <atomic>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <queue>
#include <stdexcept>

#include "biluk_internal.h"

namespace biluk {

// ---------------------------------------------------------------------------
// symbolic phase (symbolic.py:27-72)
//
// Row i is eliminated against its pivots p < i in ascending order (a min-heap;
// the reference keeps a sorted list with insort after the cursor, :51-65).
// Offering (i, j) the level lev(i,p) + lev(p,j) + 1 through pivot p, keeping
// the minimum, and never storing a level above k reproduces the reference
// pattern exactly: the same candidates are visited in the same order with the
// same integer arithmetic.  `upper` keeps, per finalized row, its (col, level)
// pairs right of the diagonal (:44-45, :70-71).
// ---------------------------------------------------------------------------
// the reference's row-merge order, row after row (each row merges the
// finished upper rows it references): kept as the cross-check of the
// row-parallel form below (BILUK_SYMBOLIC=sequential)
static int symbolic_phase_rows(int64_t n, const int32_t *rp, const int32_t *ci, int k, std::vector<int32_t> &out_rp,
                               std::vector<int32_t> &out_ci, int64_t *err_row) {
    if (k == 0) {
        // ILU(0): every entry of A has level 0 and nothing fills in -- the
        // pattern is A's, once every row is known to hold its diagonal
        for (int64_t i = 0; i < n; ++i)
            if (!std::binary_search(ci + rp[i], ci + rp[i + 1], int32_t(i))) {
                if (err_row) *err_row = i;
                return fail(BILUK_ESTRUCT, "row " + std::to_string(i) + " has no diagonal entry");
            }
        out_rp.assign(rp, rp + n + 1);
        out_ci.assign(ci, ci + rp[n]);
        return BILUK_OK;
    }
    std::vector<int32_t> lev(n, -1);
    std::vector<int64_t> up_ptr(n + 1, 0);
    std::vector<int32_t> up_col;
    std::vector<int32_t> up_lev;
    up_col.reserve(size_t(rp[n]));
    up_lev.reserve(size_t(rp[n]));
    out_rp.assign(n + 1, 0);
    out_ci.clear();
    out_ci.reserve(size_t(rp[n]) * (k > 0 ? 2 : 1));
    std::vector<int32_t> touched;
    std::vector<int32_t> heap;
    auto cmp = std::greater<int32_t>();
    for (int64_t i = 0; i < n; ++i) {
        touched.clear();
        heap.clear();
        for (int32_t t = rp[i]; t < rp[i + 1]; ++t) {
            const int32_t j = ci[t];
            lev[j] = 0;
            touched.push_back(j);
            if (j < i) heap.push_back(j);
        }
        if (lev[i] != 0) {
            for (int32_t j : touched) lev[j] = -1;
            if (err_row) *err_row = i;
            return fail(BILUK_ESTRUCT, "row " + std::to_string(i) + " has no diagonal entry");
        }
        std::make_heap(heap.begin(), heap.end(), cmp);
        while (!heap.empty()) {
            std::pop_heap(heap.begin(), heap.end(), cmp);
            const int32_t p = heap.back();
            heap.pop_back();
            const int32_t lp = lev[p];
            for (int64_t u = up_ptr[p]; u < up_ptr[p + 1]; ++u) {
                const int32_t lv = lp + up_lev[u] + 1;
                if (lv > k) continue;
                const int32_t j = up_col[u];
                const int32_t cur = lev[j];
                if (cur < 0) {
                    lev[j] = lv;
                    touched.push_back(j);
                    if (j < i) {
                        heap.push_back(j);
                        std::push_heap(heap.begin(), heap.end(), cmp);
                    }
                } else if (lv < cur) {
                    lev[j] = lv;
                }
            }
        }
        std::sort(touched.begin(), touched.end());
        for (int32_t j : touched) {
            out_ci.push_back(j);
            if (j > i) {
                up_col.push_back(j);
                up_lev.push_back(lev[j]);
            }
            lev[j] = -1;
        }
        if (out_ci.size() > size_t(INT32_MAX))
            return fail(BILUK_EUNSUPPORTED, "ILU(k) pattern exceeds 2^31 blocks");
        out_rp[i + 1] = int32_t(out_ci.size());
        up_ptr[i + 1] = int64_t(up_col.size());
    }
    return BILUK_OK;
}

// Row-parallel form.  The level of entry (i, j) is the length minus one of
// the shortest path i -> ... -> j in the graph of A whose intermediate
// vertices are all smaller than min(i, j) (the characterisation the row
// merge above computes incrementally: split any such path at its largest
// intermediate p and both halves are entries of rows i and p).  So every
// row is found on its own: breadth-first layers of path length 1 .. k+1,
// each vertex keeping the smallest possible largest-intermediate over paths
// of that length (min of max composes layer by layer); j joins the row at
// the first length whose bound is below min(i, j).  Rows are split over the
// host cores; the result is bit-identical to the row merge (tests compare
// both on grids and random patterns, and the goldens pin the reference).
int symbolic_phase(int64_t n, const int32_t *rp, const int32_t *ci, int k, std::vector<int32_t> &out_rp,
                   std::vector<int32_t> &out_ci, int64_t *err_row) {
    if (k < 0) return fail(BILUK_EARG, "fill level k must be nonnegative");
    const char *mode = std::getenv("BILUK_SYMBOLIC");
    if (k == 0 || (mode && std::string(mode) == "sequential") || n < 4096)
        return symbolic_phase_rows(n, rp, ci, k, out_rp, out_ci, err_row);
    unsigned nt = std::thread::hardware_concurrency();
    if (const char *e = std::getenv("BILUK_PLAN_THREADS")) nt = unsigned(std::max(1, std::atoi(e)));
    nt = std::max(1u, std::min(nt, 64u));
    const int64_t nblk = std::min<int64_t>(int64_t(nt) * 16, n);
    std::vector<std::vector<int32_t>> cols(nblk);          // each block's rows, concatenated
    std::vector<std::vector<int32_t>> lens(nblk);          // their lengths
    std::vector<int64_t> bad(nblk, -1);                     // first row without a diagonal
    std::atomic<int64_t> next{0};
    auto work = [&]() {
        std::vector<std::pair<int32_t, int32_t>> cur, nxt, res;   // (vertex, bound) / (vertex, length)
        for (int64_t b = next++; b < nblk; b = next++) {
            const int64_t i0 = n * b / nblk, i1 = n * (b + 1) / nblk;
            std::vector<int32_t> &out = cols[b];
            std::vector<int32_t> &ln = lens[b];
            ln.reserve(size_t(i1 - i0));
            for (int64_t i = i0; i < i1; ++i) {
                const int32_t ii = int32_t(i);
                cur.clear();
                res.clear();
                bool diag = false;
                for (int32_t t = rp[i]; t < rp[i + 1]; ++t) {
                    const int32_t j = ci[t];
                    if (j == ii) {
                        diag = true;
                        continue;
                    }
                    res.emplace_back(j, 1);
                    cur.emplace_back(j, -1);   // no intermediate yet
                }
                if (!diag) {
                    bad[b] = i;
                    break;
                }
                for (int len = 2; len <= k + 1 && !cur.empty(); ++len) {
                    nxt.clear();
                    for (const auto &vm : cur) {
                        const int32_t v = vm.first;
                        if (v >= ii) continue;   // only smaller vertices are intermediates
                        const int32_t bound = std::max(vm.second, v);
                        for (int32_t t = rp[v]; t < rp[v + 1]; ++t)
                            if (ci[t] != ii && ci[t] != v) nxt.emplace_back(ci[t], bound);
                    }
                    std::sort(nxt.begin(), nxt.end());
                    cur.clear();
                    for (size_t a = 0; a < nxt.size(); ++a)
                        if (a == 0 || nxt[a].first != nxt[a - 1].first) cur.push_back(nxt[a]);   // smallest bound
                    for (const auto &wm : cur)
                        if (wm.second < std::min(ii, wm.first)) res.emplace_back(wm.first, len);
                }
                res.emplace_back(ii, 0);
                std::sort(res.begin(), res.end());
                int32_t cnt = 0;
                for (size_t a = 0; a < res.size(); ++a)
                    if (a == 0 || res[a].first != res[a - 1].first) {
                        out.push_back(res[a].first);
                        ++cnt;
                    }
                ln.push_back(cnt);
            }
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t) pool.emplace_back(work);
    for (std::thread &t : pool) t.join();
    for (int64_t b = 0; b < nblk; ++b)
        if (bad[b] >= 0) {
            if (err_row) *err_row = bad[b];
            return fail(BILUK_ESTRUCT, "row " + std::to_string(bad[b]) + " has no diagonal entry");
        }
    int64_t total = 0;
    for (int64_t b = 0; b < nblk; ++b) total += int64_t(cols[b].size());
    if (total > int64_t(INT32_MAX)) return fail(BILUK_EUNSUPPORTED, "ILU(k) pattern exceeds 2^31 blocks");
    out_rp.assign(n + 1, 0);
    out_ci.resize(size_t(total));
    int64_t row = 0, at = 0;
    for (int64_t b = 0; b < nblk; ++b) {
        for (int32_t c : lens[b]) {
            out_rp[row + 1] = out_rp[row] + c;
            ++row;
        }
        std::copy(cols[b].begin(), cols[b].end(), out_ci.begin() + at);
        at += int64_t(cols[b].size());
        std::vector<int32_t>().swap(cols[b]);
    }
    return BILUK_OK;
}

// ---------------------------------------------------------------------------
// Eq. (4) level sets (trisolve.py:98-118): l(i) = 1 + max over referenced rows;
// lower operands scanned forward, upper operands in reverse (:109).
// ---------------------------------------------------------------------------
void level_schedule(int64_t m, const int64_t *rp, const int64_t *ci, bool upper, int64_t *lev, int64_t *nlev) {
    int64_t mx = 0;
    for (int64_t s = 0; s < m; ++s) {
        const int64_t i = upper ? m - 1 - s : s;
        int64_t best = 0;
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) best = std::max(best, lev[ci[t]]);
        lev[i] = best + 1;
        mx = std::max(mx, lev[i]);
    }
    *nlev = mx;
}

namespace {

// Tiles of one sweep: rows grouped by block level, ascending row index inside
// a level.  On stencil matrices the dependencies of consecutive rows of a
// level are then consecutive rows of earlier levels, so a warp's dependency
// loads coalesce.  Tiles never straddle two levels, so every dependency of a
// tile lives in a strictly earlier tile -- the deadlock-freedom argument of
// the persistent sweep.
void build_sweep(const Plan &p, bool upper, const std::vector<int32_t> &lev, int32_t nlev, Sweep &sw,
                 const Sweep *lower_sweep) {
    const int R = rows_per_tile(p.bs);
    const int64_t n = p.n;
    auto nslot = [&](int64_t i) -> int32_t {
        return upper ? p.p_rp[i + 1] - p.p_diag[i] - 1 : p.p_diag[i] - p.p_rp[i];
    };
    auto first_slot = [&](int64_t i) -> int32_t { return upper ? p.p_diag[i] + 1 : p.p_rp[i]; };
    std::vector<int64_t> cnt(nlev + 2, 0);
    for (int64_t i = 0; i < n; ++i) cnt[lev[i]]++;
    std::vector<int64_t> start(nlev + 2, 0);
    for (int l = 1; l <= nlev + 1; ++l) start[l] = start[l - 1] + cnt[l - 1];
    std::vector<int32_t> order(n);
    {
        std::vector<int64_t> cur(start);
        for (int64_t i = 0; i < n; ++i) order[cur[lev[i]]++] = int32_t(i);
    }
    sw.tile_rows.clear();
    sw.meta.clear();
    sw.pos.assign(n, -1);
    sw.rec_total = 0;
    sw.max_slots = 0;
    sw.max_rec = 0;
    for (int l = 1; l <= nlev; ++l) {
        auto b = order.begin() + start[l], e = order.begin() + start[l] + cnt[l];
        for (auto it = b; it < e; it += R) {
            const int64_t take = std::min<int64_t>(R, e - it);
            int32_t S = 0;
            // probes: an ancestor one and two levels back (positions of earlier levels are known);
            // U' tiles without such an ancestor wait on a y value of the L sweep instead
            int32_t probe1 = -1, probe2 = -1, ypos = -1;
            for (int64_t q = 0; q < take; ++q) {
                const int64_t i = it[q];
                sw.pos[i] = int32_t(sw.tile_rows.size());
                sw.tile_rows.push_back(int32_t(i));
                S = std::max(S, nslot(i));
                if (lower_sweep) ypos = std::max(ypos, lower_sweep->pos[i]);
                for (int32_t t = first_slot(i), e = first_slot(i) + nslot(i); t < e; ++t) {
                    const int32_t j = p.p_ci[t];
                    if (lev[j] != l - 1) continue;
                    probe1 = std::max(probe1, sw.pos[j]);
                    if (lower_sweep) ypos = std::max(ypos, lower_sweep->pos[j]);
                    for (int32_t u = first_slot(j), f = first_slot(j) + nslot(j); u < f; ++u)
                        if (lev[p.p_ci[u]] == l - 2) probe2 = std::max(probe2, sw.pos[p.p_ci[u]]);
                }
            }
            if (upper && ypos >= 0) {
                if (probe1 < 0) probe1 = -(ypos + 2);
                if (probe2 < 0) probe2 = -(ypos + 2);
            }
            for (int64_t q = take; q < R; ++q) sw.tile_rows.push_back(-1);
            TileMeta m{};
            m.off128 = uint32_t(sw.rec_total / 128);
            m.nslot = S;
            m.level = l;
            m.probe[0] = probe1;
            m.probe[1] = probe2;
            sw.meta.push_back(m);
            const int64_t bytes = rec_bytes(p.bs, S, upper);
            sw.rec_total += bytes;
            sw.max_slots = std::max(sw.max_slots, S);
            sw.max_rec = std::max(sw.max_rec, bytes);
        }
    }
    sw.ntiles = int64_t(sw.meta.size());
}

}  // namespace

int plan_analyse(Plan &p, int32_t bs, int64_t n, const int64_t *rp, const int64_t *ci, int32_t k, int64_t *err_row) {
    if (bs < 1 || bs > 8) return fail(BILUK_EUNSUPPORTED, "block size must be in 1..8 on this path");
    if (n < 0) return fail(BILUK_ESTRUCT, "negative dimension");
    if (k < 0) return fail(BILUK_EARG, "fill level k must be nonnegative");
    if (n >= INT32_MAX || rp[n] >= INT32_MAX) return fail(BILUK_EUNSUPPORTED, "matrix exceeds 2^31 blocks");
    p.bs = bs;
    p.n = n;
    p.k = k;
    p.nnzA = rp[n];
    // structural validation (sparse.py:35-52)
    if (rp[0] != 0) return fail(BILUK_ESTRUCT, "row_ptr must start at 0");
    p.a_rp.resize(n + 1);
    p.a_ci.resize(p.nnzA);
    for (int64_t i = 0; i < n; ++i) {
        if (rp[i + 1] < rp[i]) return fail(BILUK_ESTRUCT, "row_ptr must be nondecreasing");
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
            if (ci[t] < 0 || ci[t] >= n) return fail(BILUK_ESTRUCT, "column index out of range");
            if (t > rp[i] && ci[t] <= ci[t - 1])
                return fail(BILUK_ESTRUCT, "column indices must increase strictly within a row");
            p.a_ci[t] = int32_t(ci[t]);
        }
    }
    for (int64_t i = 0; i <= n; ++i) p.a_rp[i] = int32_t(rp[i]);

    const auto t_sym = std::chrono::steady_clock::now();
    int rc = symbolic_phase(n, p.a_rp.data(), p.a_ci.data(), k, p.p_rp, p.p_ci, err_row);
    if (std::getenv("BILUK_PLAN_TIMING"))
        std::fprintf(stderr, "[plan] symbolic %.3f s\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t_sym).count());
    if (rc != BILUK_OK) return rc;
    p.nnzP = p.p_rp[n];
    p.p_diag.resize(n);
    p.nL = p.nU = 0;
    p.max_row_len = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t *b = p.p_ci.data() + p.p_rp[i], *e = p.p_ci.data() + p.p_rp[i + 1];
        const int32_t *d = std::lower_bound(b, e, int32_t(i));
        p.p_diag[i] = int32_t(d - p.p_ci.data());
        p.nL += d - b;
        p.nU += e - d - 1;
        p.max_row_len = std::max<int32_t>(p.max_row_len, int32_t(e - b));
    }
    // A slot -> P' slot (materialize, factor.py:107-118); P' contains A by construction
    p.a2p.resize(p.nnzA);
    for (int64_t i = 0; i < n; ++i) {
        int32_t q = p.p_rp[i];
        for (int32_t t = p.a_rp[i]; t < p.a_rp[i + 1]; ++t) {
            while (p.p_ci[q] != p.a_ci[t]) ++q;
            p.a2p[t] = q;
        }
    }
    // block level sets of L (forward) and U' (reverse)
    p.lev_L.assign(n, 0);
    p.lev_U.assign(n, 0);
    p.nlev_L = p.nlev_U = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t best = 0;
        for (int32_t t = p.p_rp[i]; t < p.p_diag[i]; ++t) best = std::max(best, p.lev_L[p.p_ci[t]]);
        p.lev_L[i] = best + 1;
        p.nlev_L = std::max(p.nlev_L, best + 1);
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        int32_t best = 0;
        for (int32_t t = p.p_diag[i] + 1; t < p.p_rp[i + 1]; ++t) best = std::max(best, p.lev_U[p.p_ci[t]]);
        p.lev_U[i] = best + 1;
        p.nlev_U = std::max(p.nlev_U, best + 1);
    }
    // factorization order: rows by L level (row i needs every pivot row p < i of its L pattern)
    p.fptr.assign(p.nlev_L + 1, 0);
    for (int64_t i = 0; i < n; ++i) p.fptr[p.lev_L[i]]++;
    for (int l = 1; l <= p.nlev_L; ++l) p.fptr[l] += p.fptr[l - 1];
    p.forder.resize(n);
    {
        std::vector<int64_t> cur(p.nlev_L + 1, 0);
        for (int l = 1; l <= p.nlev_L; ++l) cur[l] = p.fptr[l - 1];
        for (int64_t i = 0; i < n; ++i) p.forder[cur[p.lev_L[i]]++] = int32_t(i);
    }
    return BILUK_OK;
}

// tile layout of the level-order engine (engine 0)
int plan_tiles(Plan &p) {
    build_sweep(p, false, p.lev_L, p.nlev_L, p.sl, nullptr);
    build_sweep(p, true, p.lev_U, p.nlev_U, p.su, &p.sl);
    // tiles per combined level: L levels 1..nlev_L, then U' levels nlev_L+1..
    p.lvl_tiles.assign(size_t(p.nlev_L) + p.nlev_U + 2, 0);
    for (const TileMeta &m : p.sl.meta) p.lvl_tiles[m.level]++;
    for (const TileMeta &m : p.su.meta) p.lvl_tiles[p.nlev_L + m.level]++;
    if ((p.sl.rec_total / 128) >= (int64_t(1) << 32) || (p.su.rec_total / 128) >= (int64_t(1) << 32))
        return fail(BILUK_EUNSUPPORTED, "factor records exceed 512 GB");
    return BILUK_OK;
}

// structural validation of a CSR / BSR index structure (sparse.py:35-52)
int validate_bsr(int64_t n, int64_t ncols, const int64_t *rp, const int64_t *ci) {
    if (n < 0 || ncols < 0) return fail(BILUK_ESTRUCT, "negative dimension");
    if (rp[0] != 0) return fail(BILUK_ESTRUCT, "row_ptr must have num_rows+1 entries starting at 0");
    for (int64_t i = 0; i < n; ++i) {
        if (rp[i + 1] < rp[i]) return fail(BILUK_ESTRUCT, "row_ptr must be nondecreasing");
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
            if (ci[t] < 0 || ci[t] >= ncols) return fail(BILUK_ESTRUCT, "column index out of range");
            if (t > rp[i] && ci[t] <= ci[t - 1])
                return fail(BILUK_ESTRUCT, "column indices must increase strictly within a row");
        }
    }
    return BILUK_OK;
}

// SpMV operator: sliced-ELL tiles of R consecutive block rows
int op_analyse(Op &o, int32_t bs, int64_t n, int64_t ncols, const int64_t *rp, const int64_t *ci) {
    if (bs < 1 || bs > 8) return fail(BILUK_EUNSUPPORTED, "block size must be in 1..8 on this path");
    int rc = validate_bsr(n, ncols, rp, ci);
    if (rc != BILUK_OK) return rc;
    if (n >= INT32_MAX || ncols >= INT32_MAX || rp[n] >= INT32_MAX)
        return fail(BILUK_EUNSUPPORTED, "matrix exceeds 2^31 blocks");
    o.bs = bs;
    o.n = n;
    o.ncols = ncols;
    o.nnz = rp[n];
    o.rp.resize(n + 1);
    o.ci.resize(o.nnz);
    for (int64_t i = 0; i <= n; ++i) o.rp[i] = int32_t(rp[i]);
    for (int64_t t = 0; t < o.nnz; ++t) o.ci[t] = int32_t(ci[t]);
    const int R = rows_per_tile(bs);
    o.ntiles = (n + R - 1) / R;
    o.meta.resize(o.ntiles);
    o.rec_total = 0;
    for (int64_t t = 0; t < o.ntiles; ++t) {
        int32_t S = 0;
        for (int64_t i = t * R; i < std::min<int64_t>(n, (t + 1) * R); ++i) S = std::max(S, o.rp[i + 1] - o.rp[i]);
        o.meta[t] = TileMeta{};
        o.meta[t].off128 = uint32_t(o.rec_total / 128);
        o.meta[t].nslot = S;
        o.meta[t].probe[0] = o.meta[t].probe[1] = -1;
        o.rec_total += ell_bytes(bs, S);
    }
    if (o.rec_total / 128 >= (int64_t(1) << 32)) return fail(BILUK_EUNSUPPORTED, "operator exceeds 512 GB");
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        uint64_t at = off;
        off += (bytes + 255) & ~uint64_t(255);
        return at;
    };
    o.off.rp = take(4 * (n + 1));
    o.off.ci = take(4 * o.nnz);
    o.off.meta = take(sizeof(TileMeta) * o.ntiles);
    o.off.rec = take(o.rec_total);
    o.off.total = off;
    return BILUK_OK;
}

void plan_layout(Plan &p, int num_sms, size_t smem_per_sm) {
    // sweep launch: one CTA per SM holding as many warps as the double-buffered
    // tile ring allows (each warp owns `stages` stage buffers of the largest record)
    p.num_sms = num_sms;
    if (p.engine == 2) {
        p.sweep_ctas = p.gs.P;
        p.sweep_warps = 12 + 1 + 3;   // compute groups, producer, halo warps (gsweep.cu)
        p.sweep_stages = p.gs.kslots;
        p.stage_bytes = p.gs.slot_bytes;
    } else if (p.engine == 1) {
        p.sweep_ctas = p.ps.P;
        p.sweep_warps = p.ps.groups * p.ps.nthreads / 32 + p.ps.nprod;   // compute groups + producers
        p.sweep_stages = PS_KSLOTS;
        p.stage_bytes = p.ps.max_rec;
    } else {
    p.stage_bytes = std::max<int64_t>(128, std::max(p.sl.max_rec, p.su.max_rec));
    const size_t budget = smem_per_sm > 8192 ? smem_per_sm - 4096 : smem_per_sm;
    int stages = 2;
    int warps = int(budget / (size_t(stages) * p.stage_bytes + 16 * stages));
    if (warps < 1) {
        stages = 1;
        warps = int(budget / (size_t(p.stage_bytes) + 16));
    }
    warps = std::max(1, std::min(warps, 8));   // <= 256 threads: the kernel keeps 255 registers
    p.sweep_stages = stages;
    p.sweep_warps = warps;
    p.sweep_ctas = num_sms;
    }

    const int64_t bs2 = int64_t(p.bs) * p.bs;
    uint64_t o = 0;
    auto take = [&](uint64_t bytes) {
        uint64_t at = o;
        o += (bytes + 255) & ~uint64_t(255);
        return at;
    };
    p.off.p_rp = take(4 * (p.n + 1));
    p.off.p_ci = take(4 * p.nnzP);
    p.off.p_diag = take(4 * p.n);
    p.off.a2p = take(4 * p.nnzA);
    p.off.forder = take(4 * p.n);
    p.off.pvals = take(8 * p.nnzP * bs2);
    p.off.dinv = take(8 * p.n * bs2);
    const int R = rows_per_tile(p.bs);
    p.off.sl_rows = take(4 * p.sl.ntiles * R);
    p.off.sl_meta = take(sizeof(TileMeta) * p.sl.ntiles);
    p.off.sl_rec = take(p.sl.rec_total);
    p.off.su_rows = take(4 * p.su.ntiles * R);
    p.off.su_meta = take(sizeof(TileMeta) * p.su.ntiles);
    p.off.su_rec = take(p.su.rec_total);
    p.off.pos_l = take(4 * p.n);
    p.off.pos_u = take(4 * p.n);
    p.off.y_t = take(8 * plan_npos(p) * plan_vs(p));   // rows at L positions
    p.off.x_t = take(8 * plan_npos(p) * plan_vs(p));   // rows at U' positions
    p.off.lvl_tiles = take(4 * p.lvl_tiles.size());
    p.off.lvl_cnt = take(4 * p.lvl_tiles.size());
    p.off.status = take(sizeof(DevStatus));
    p.off.ps_rec = take(p.ps.rec_total);
    p.off.ps_info = take(sizeof(PRecInfo) * p.ps.rec.size());
    p.off.ps_part = take(4 * p.ps.part_rec.size());
    p.off.ps_idx = take(4 * p.ps.idx.size());
    p.off.ps_vmap = take(4 * p.ps.vmap.size());
    const bool ps_on = p.engine == 1;
    p.off.ps_posl = take(ps_on ? 4 * p.n : 0);                               // L position -> row
    p.off.ps_bperm = take(ps_on ? 8 * p.n * p.bs + 16 : 0);                  // b in L-position order (packed)
    p.off.ps_yu = take(ps_on ? 8 * p.n * p.bs + 16 : 0);                     // y in U'-position order (packed)
    const bool gs_on = p.engine == 2;
    p.off.gs_part = take(gs_on ? sizeof(GPart) * p.gs.part.size() : 0);
    p.off.gs_rec = take(gs_on ? sizeof(GRec) * p.gs.rec.size() : 0);
    p.off.gs_lo = take(gs_on ? 4 * p.gs.rec_lo.size() : 0);
    p.off.gs_cols = take(gs_on ? 4 * p.gs.cols.size() : 0);
    p.off.gs_stream = take(gs_on ? uint64_t(p.gs.stream_bytes) : 0);
    p.off.gs_y = take(gs_on ? 8 * p.n * p.bs : 0);                          // y in natural order
    p.off.total = o;
}

}  // namespace biluk
