// Host planner of the partitioned sweep (the apply engine).
//
// Replaces the execution side of build_level_schedule / _pack_level
// (trisolve.py:83-118): the reference packs every level of each triangle
// into one gather/reduceat/scatter pass per level (trisolve.py:121-145); here
// the same level sets (global block levels of L and U', bit-exact with
// level_schedule) order the rows INSIDE contiguous row ranges ("parts"), one
// CTA per part, and the records a CTA streams are laid out back to back.
// Integer work only; the values are packed on the device (ppack_kernel).
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>

#include "biluk_internal.h"

namespace biluk {

namespace {

inline int64_t a16(int64_t x) { return (x + 15) & ~int64_t(15); }

// bytes of a record with the given shape (layout: biluk_internal.h)
// int32 words of a record's index section: header, iarr, desc (int16 entries,
// two per word), gpos
inline int64_t rec_desc_words(int nrows, int S) { return (int64_t(S) * nrows + 1) / 2; }
inline int64_t rec_index_words(int nrows, int S, int nglob, bool upper) {
    (void)upper;
    return int64_t(sizeof(PRecHdr) / 4) + int64_t(nrows) + rec_desc_words(nrows, S) + nglob;
}
inline int64_t rec_vals_off(int nrows, int S, int nglob, bool upper) {
    return a16(4 * rec_index_words(nrows, S, nglob, upper));
}
inline int64_t rec_total_bytes(int bs2, int nrows, int S, int nglob, bool upper) {
    return a16(rec_vals_off(nrows, S, nglob, upper) + 8 * int64_t(bs2) * nrows * (S + (upper ? 1 : 0)));
}
// shared-memory footprint: the streamed bytes, the inputs (ps_in_bytes: bs
// doubles per row) and the fetched dependencies (bs doubles each, exact)
inline int64_t rec_foot_bytes(int bs2, int vs, int nrows, int S, int nglob, bool upper) {
    const int bs = int(std::lround(std::sqrt(double(bs2))));
    (void)vs;
    return rec_total_bytes(bs2, nrows, S, nglob, upper) + ps_in_bytes(bs, nrows) + a16(int64_t(nglob) * bs * 8);
}

inline int32_t nslot_of(const Plan &p, int64_t i, bool upper) {
    return upper ? p.p_rp[i + 1] - p.p_diag[i] - 1 : p.p_diag[i] - p.p_rp[i];
}
inline int32_t first_slot_of(const Plan &p, int64_t i, bool upper) { return upper ? p.p_diag[i] + 1 : p.p_rp[i]; }

// streamed bytes of row i in both sweeps (balancing weight)
inline int64_t row_weight(const Plan &p, int64_t i) {
    const int64_t s = nslot_of(p, i, false) + nslot_of(p, i, true), bs2 = int64_t(p.bs) * p.bs;
    return (s + 1) * bs2 * 8 + 8 * s + 16 * p.bs + 16;
}

// contiguous row ranges of (nearly) equal streamed bytes
void partition_contiguous(const Plan &p, int P, Partition &pt) {
    const int64_t n = p.n;
    std::vector<int64_t> cum(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) cum[i + 1] = cum[i] + row_weight(p, i);
    std::vector<int32_t> ptr(P + 1, 0);
    ptr[P] = int32_t(n);
    for (int c = 1; c < P; ++c) {
        const int64_t target = (cum[n] * c + P / 2) / P;
        int64_t r = std::lower_bound(cum.begin(), cum.end(), target) - cum.begin();
        r = std::max<int64_t>(r, ptr[c - 1]);
        ptr[c] = int32_t(std::min<int64_t>(r, n));
    }
    pt.P = P;
    pt.kind = 0;
    pt.part_of.resize(n);
    for (int c = 0; c < P; ++c)
        for (int32_t i = ptr[c]; i < ptr[c + 1]; ++i) pt.part_of[i] = c;
}

// structured-grid columns: (y, z) blocks spanning every x of a natural-order grid
void partition_columns(const Plan &p, int P, const int64_t g[3], Partition &pt) {
    const int64_t nx = g[0], ny = g[1], nz = g[2];
    // as many parts as allowed whose columns fit one record per level (a part
    // of more than 128 columns splits each level into two records: twice the
    // chain); among those, about twice as many parts along z as along y,
    // ties to the larger pz (128^3 ILU(0) sweep: 12x12 558 us, 11x13 547,
    // 9x16 540.5, 8x18 537.7 over three runs each; 10x14 -- 130 columns per
    // part -- 741)
    int best_y = 1, best_z = 1;
    double best = -1e300;
    for (int pz = 1; pz <= std::min<int64_t>(P, nz); ++pz) {
        const int py = int(std::min<int64_t>(ny, P / pz));
        if (py < 1) continue;
        const int64_t cols = ((ny + py - 1) / py) * ((nz + pz - 1) / pz);
        const double score = (cols <= 128 ? 1e9 : 0.0) + double(py) * pz - 3.0 * std::abs(double(pz) - 2.0 * py);
        if (score >= best) {
            best = score;
            best_y = py;
            best_z = pz;
        }
    }
    if (const char *env = std::getenv("BILUK_SPLIT")) {   // diagnostics: parts along y,z
        int sy = 0, sz = 0;
        if (std::sscanf(env, "%d,%d", &sy, &sz) == 2 && sy >= 1 && sz >= 1 && sy <= ny && sz <= nz && sy * sz <= P) {
            best_y = sy;
            best_z = sz;
        }
    }
    pt.P = best_y * best_z;
    pt.kind = 1;
    pt.grid[0] = nx;
    pt.grid[1] = ny;
    pt.grid[2] = nz;
    pt.split[0] = best_y;
    pt.split[1] = best_z;
    pt.part_of.resize(p.n);
    for (int64_t k = 0; k < nz; ++k) {
        const int cz = int(k * best_z / nz);
        for (int64_t j = 0; j < ny; ++j) {
            const int c = cz * best_y + int(j * best_y / ny);
            const int64_t r = (k * ny + j) * nx;
            for (int64_t i = 0; i < nx; ++i) pt.part_of[r + i] = c;
        }
    }
}

// rows of every part (ascending) and their position bases
void partition_finish(Partition &pt) {
    pt.rows.assign(pt.P, {});
    std::vector<int64_t> cnt(pt.P, 0);
    for (int32_t c : pt.part_of) cnt[c]++;
    for (int c = 0; c < pt.P; ++c) pt.rows[c].reserve(cnt[c]);
    for (size_t i = 0; i < pt.part_of.size(); ++i) pt.rows[pt.part_of[i]].push_back(int32_t(i));
    pt.base.assign(pt.P + 1, 0);
    for (int c = 0; c < pt.P; ++c) pt.base[c + 1] = pt.base[c] + int32_t(cnt[c]);
}

// a part's rows in (level, row) order
void part_order(const std::vector<int32_t> &lev, const std::vector<int32_t> &rows, std::vector<int32_t> &ord) {
    ord = rows;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return lev[a] < lev[b]; });
}

// run f(c) for c in [0, P) on the host's cores (the parts are independent)
template <class F>
void parallel_parts(int P, F f) {
    unsigned nt = std::thread::hardware_concurrency();
    if (const char *e = std::getenv("BILUK_PLAN_THREADS")) nt = unsigned(std::max(1, std::atoi(e)));
    nt = std::max(1u, std::min<unsigned>(nt, unsigned(P)));
    if (nt <= 1) {
        for (int c = 0; c < P; ++c) f(c);
        return;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t)
        pool.emplace_back([&]() {
            for (int c = next++; c < P; c = next++) f(c);
        });
    for (std::thread &t : pool) t.join();
}

// the records of part c (both sweeps): the level-ordered rows cut into
// chunks of <= nthreads rows of one level under the footprint caps; offsets
// (record bytes, index words, value-map entries) relative to the part
struct PartRecords {
    std::vector<PRecInfo> rec;
    std::vector<int32_t> idx, vmap;
    int64_t rec_total = 0, max_rec = 0, max_glob = 0, nglob_total = 0;
    int32_t nl = 0;   // L records
    int rc = BILUK_OK;
    std::string msg;
};

void build_part_records(const Plan &p, const Partition &pt, const std::vector<int32_t> &ordLc,
                        const std::vector<int32_t> &ordUc, int c, PartRecords &out) {
    const PSweep &ps = p.ps;
    const int bs = p.bs, bs2 = bs * bs, vs = ps_vec_stride(bs);
    const int32_t mask = ps.ring - 1;
    std::vector<int32_t> gl;     // a record's deduplicated dependency positions
    std::vector<int32_t> nfar;   // per row of a level group: dependencies outside the ring
    struct Chunk {
        size_t a, e;           // rows ord[a, e) of one level
        int64_t lend;          // ring sequence number just past the level
        int S;
        int64_t far;           // dependencies outside the ring (upper bound, not deduplicated)
    };
    std::vector<Chunk> chunks;
    {
        const int32_t b0 = pt.base[c];
        const int32_t m = pt.base[c + 1] - b0;
        for (int pass = 0; pass < 2; ++pass) {
            const bool up = pass == 1;
            const std::vector<int32_t> &ord = up ? ordUc : ordLc;
            const std::vector<int32_t> &lev = up ? p.lev_U : p.lev_L;
            const std::vector<int32_t> &pos = up ? ps.posU : ps.posL;
            const int32_t seq_base = up ? m : 0;   // ring sequence continues from the L sweep
            const size_t rec_begin = out.rec.size();
            // a dependency j of a row of a level ending at sequence `lend` is on
            // chip iff it is in this part and the level's own writes cannot have
            // recycled its ring slot
            auto in_ring = [&](int32_t j, int64_t lend) {
                return pt.part_of[j] == c && seq_base + int64_t(pos[j] - b0) >= lend - ps.ring;
            };
            // ---- chunks: <= nthreads rows of one level under the caps
            chunks.clear();
            size_t g0 = 0;
            while (g0 < ord.size()) {
                size_t ge = g0;
                while (ge < ord.size() && lev[ord[ge]] == lev[ord[g0]]) ++ge;
                const int64_t lend = seq_base + int64_t(ge);
                nfar.assign(ge - g0, 0);
                for (size_t q = g0; q < ge; ++q) {
                    const int32_t i = ord[q];
                    const int32_t fs = first_slot_of(p, i, up), ns = nslot_of(p, i, up);
                    for (int32_t s2 = fs; s2 < fs + ns; ++s2) nfar[q - g0] += in_ring(p.p_ci[s2], lend) ? 0 : 1;
                }
                size_t a = g0;
                while (a < ge) {
                    size_t e = a;
                    int S = 0;
                    int64_t far = 0;
                    while (e < ge && int64_t(e - a) < ps.nthreads) {
                        const int32_t i = ord[e];
                        const int S2 = std::max<int>(S, nslot_of(p, i, up));
                        const int64_t far2 = far + nfar[e - g0];
                        const int nr = int(e - a + 1);
                        if (e > a && (rec_foot_bytes(bs2, vs, nr, S2, int(far2), up) > ps.rec_cap || far2 > ps.glob_cap))
                            break;
                        S = S2;
                        far = far2;
                        ++e;
                    }
                    chunks.push_back({a, e, lend, S, far});
                    a = e;
                }
                g0 = ge;
            }
            // ---- records: one chunk each (pairing two whole levels per record
            // was measured neutral to slower)
            for (size_t ci0 = 0; ci0 < chunks.size();) {
                const size_t a = chunks[ci0].a, e = chunks[ci0].e;
                const int nr = int(e - a);
                const int S = chunks[ci0].S;
                auto lend_of = [&](size_t) { return chunks[ci0].lend; };
                gl.clear();
                for (size_t q = a; q < e; ++q) {
                    const int32_t i = ord[q];
                    const int32_t fs = first_slot_of(p, i, up), ns = nslot_of(p, i, up);
                    for (int32_t s2 = fs; s2 < fs + ns; ++s2)
                        if (!in_ring(p.p_ci[s2], lend_of(q))) gl.push_back(pos[p.p_ci[s2]]);
                }
                std::sort(gl.begin(), gl.end());
                gl.erase(std::unique(gl.begin(), gl.end()), gl.end());
                const int nglob = int(gl.size());
                const int64_t foot = rec_foot_bytes(bs2, vs, nr, S, nglob, up);
                if (nglob > ps.glob_cap || foot > ps.data_ring / 4 || foot >= (int64_t(1) << 31)) {   // half a producer's half ring
                    out.rc = BILUK_EUNSUPPORTED;
                    out.msg = "a block row is too long for the partitioned sweep";
                    return;
                }
                const int32_t lvl = lev[ord[a]];
                PRecInfo info{};
                info.nrows = nr;
                info.S = S;
                info.level = lvl * 2 + (up ? 1 : 0);
                info.nglob = nglob;
                info.pos0 = int32_t(b0 + int32_t(a));
                info.bytes = uint32_t(rec_total_bytes(bs2, nr, S, nglob, up));
                info.foot = uint32_t(foot);
                info.idx_words = uint32_t(rec_index_words(nr, S, nglob, up));
                info.off = uint64_t(out.rec_total);
                info.idx_off = uint64_t(out.idx.size());
                info.vmap_off = int64_t(out.vmap.size());
                out.rec_total += info.bytes;
                out.max_rec = std::max<int64_t>(out.max_rec, foot);
                out.max_glob = std::max<int64_t>(out.max_glob, nglob);
                out.nglob_total += nglob;
                PRecHdr h{};
                h.nrows = nr;
                h.S = S;
                h.nglob = nglob;
                h.flags = (up ? 1 : 0) | (nr << 1) | (lvl << 10);
                h.seq0 = int32_t(seq_base + int32_t(a));
                h.pos0 = int32_t(b0 + int32_t(a));
                h.vals_off = int32_t(rec_vals_off(nr, S, nglob, up));
                h.in_off = int32_t(info.bytes);
                const size_t base = out.idx.size();
                out.idx.resize(base + size_t(a16(4 * int64_t(info.idx_words)) / 4), 0);   // 16-byte aligned sections
                std::memcpy(out.idx.data() + base, &h, sizeof(h));
                int32_t *w = out.idx.data() + base + sizeof(PRecHdr) / 4;
                for (int q = 0; q < nr; ++q) w[q] = up ? ord[a + q] : ps.posU[ord[a + q]];
                w += nr;
                int16_t *desc = reinterpret_cast<int16_t *>(w);
                int32_t *gpos = w + rec_desc_words(nr, S);
                for (int t = 0; t < nglob; ++t) gpos[t] = gl[t];
                const size_t vbase = out.vmap.size();
                out.vmap.resize(vbase + size_t(S) * nr, -1);
                for (int q = 0; q < nr; ++q) {
                    const int32_t i = ord[a + q];
                    const int32_t fs = first_slot_of(p, i, up), ns = nslot_of(p, i, up);
                    for (int s2 = 0; s2 < S; ++s2) {
                        int32_t d = ps.ring;   // zero slot
                        if (s2 < ns) {
                            const int32_t j = p.p_ci[fs + s2];
                            if (in_ring(j, lend_of(a + q))) {
                                d = int32_t((seq_base + int64_t(pos[j] - b0)) & mask);
                            } else {
                                const int64_t at = std::lower_bound(gl.begin(), gl.end(), pos[j]) - gl.begin();
                                d = -int32_t(at) - 1;   // fetched dependency `at`
                            }
                            out.vmap[vbase + size_t(s2) * nr + q] = fs + s2;
                        }
                        desc[int64_t(s2) * nr + q] = int16_t(d);   // ring slot <= ring, or -(fetched + 1) >= -glob_cap
                    }
                }
                out.rec.push_back(info);
                ++ci0;
            }
            if (!up) out.nl = int32_t(out.rec.size() - rec_begin);
        }
    }
}

}  // namespace

void partition_grid_columns(const Plan &p, int P, const int64_t g[3], Partition &pt) { partition_columns(p, P, g, pt); }

// ---------------------------------------------------------------------------
// Natural-order structured grid (nx, ny, nz) behind the block pattern of A, if
// any: the offsets 1, nx and nx*ny must each occur in >= n/4 rows.  Only the
// partition's QUALITY depends on this guess -- any row -> part assignment is
// correct, because every CTA walks its rows in global level order.
// ---------------------------------------------------------------------------
bool detect_grid(const Plan &p, int64_t g[3]) {
    const int64_t n = p.n;
    if (n < 8) return false;
    std::vector<int64_t> offs;
    offs.reserve(size_t(p.nnzA));
    for (int64_t i = 0; i < n; ++i)
        for (int32_t t = p.a_rp[i]; t < p.a_rp[i + 1]; ++t)
            if (p.a_ci[t] > i) offs.push_back(p.a_ci[t] - i);
    std::sort(offs.begin(), offs.end());
    std::vector<std::pair<int64_t, int64_t>> freq;   // offset, count
    for (size_t a = 0; a < offs.size();) {
        size_t b = a;
        while (b < offs.size() && offs[b] == offs[a]) ++b;
        if (int64_t(b - a) * 4 >= n) freq.emplace_back(offs[a], int64_t(b - a));
        a = b;
    }
    auto has = [&](int64_t o) {
        for (auto &f : freq)
            if (f.first == o) return true;
        return false;
    };
    if (!has(1)) return false;
    for (auto &fx : freq) {
        const int64_t nx = fx.first;
        if (nx < 2 || n % nx) continue;
        for (auto it = freq.rbegin(); it != freq.rend(); ++it) {
            const int64_t nxy = it->first;
            if (nxy <= nx || nxy % nx || n % nxy) continue;
            g[0] = nx;
            g[1] = nxy / nx;
            g[2] = n / nxy;
            return true;
        }
        // a 2-D grid: nx and n / nx
        g[0] = nx;
        g[1] = n / nx;
        g[2] = 1;
        return true;
    }
    return false;
}

// ---------------------------------------------------------------------------
// Cost model used to choose the partition: a level-group-granular simulation
// of the sweeps.  A level group of a part starts when the part's previous
// group is done and every cross-part dependency has been published + HOP; it
// takes TAU per record plus its streamed bytes at the per-SM rate.  The apply
// is at least the streamed bytes over the HBM rate.
// ---------------------------------------------------------------------------
double psweep_estimate_us(const Plan &p, const Partition &pt) {
    const double HOP = 1.0, TAU = 0.45, BW_SM = 80e3, BW_HBM = 6.0e6;   // us, bytes/us
    const int64_t n = p.n, bs2 = int64_t(p.bs) * p.bs;
    if (n == 0) return 0.0;
    const int P = pt.P;
    std::vector<double> finL(n, 0.0), finU(n, 0.0), part_l_end(P, 0.0);
    std::vector<int32_t> ord;
    double total_bytes = 0;
    double end = 0;
    // parts in an order in which every cross-part dependency is already timed:
    // L by the smallest row, U' by the largest (a part's rows may interleave
    // with others' -- fall back to sweeping the rows in level order globally)
    for (int pass = 0; pass < 2; ++pass) {
        const bool up = pass == 1;
        const std::vector<int32_t> &lev = up ? p.lev_U : p.lev_L;
        std::vector<double> &fin = up ? finU : finL;
        const int32_t nlev = up ? p.nlev_U : p.nlev_L;
        // rows bucketed by level; within a level, per part: group start/end
        std::vector<std::vector<int32_t>> bylev(nlev + 1);
        for (int64_t i = 0; i < n; ++i) bylev[lev[i]].push_back(int32_t(i));
        std::vector<double> t(P, 0.0);
        for (int c = 0; c < P; ++c) t[c] = up ? part_l_end[c] : 0.0;
        std::vector<double> ready(P), bytes(P);
        std::vector<int32_t> rows_in(P, 0);
        for (int32_t l = 1; l <= nlev; ++l) {
            for (int32_t i : bylev[l]) {
                const int c = pt.part_of[i];
                if (rows_in[c] == 0) {
                    ready[c] = t[c];
                    bytes[c] = 0;
                }
                rows_in[c]++;
                const int32_t fs = first_slot_of(p, i, up), ns = nslot_of(p, i, up);
                for (int32_t s = fs; s < fs + ns; ++s) {
                    const int32_t j = p.p_ci[s];
                    if (pt.part_of[j] != c) ready[c] = std::max(ready[c], fin[j] + HOP);
                }
                bytes[c] += double(ns + (up ? 1 : 0)) * bs2 * 8 + 4 * ns + 16 * p.bs;
            }
            for (int32_t i : bylev[l]) {
                const int c = pt.part_of[i];
                if (rows_in[c] > 0) {
                    const double recs = std::ceil(double(rows_in[c]) / 128.0);
                    t[c] = ready[c] + recs * TAU + bytes[c] / BW_SM;
                    total_bytes += bytes[c];
                    rows_in[c] = 0;
                }
                fin[i] = t[c];
            }
        }
        for (int c = 0; c < P; ++c) {
            if (!up) part_l_end[c] = t[c];
            end = std::max(end, t[c]);
        }
    }
    return std::max(end, total_bytes / BW_HBM);
}

// ---------------------------------------------------------------------------
// Build the records of both sweeps for P parts.
// ---------------------------------------------------------------------------
int plan_psweep(Plan &p, int num_sms, size_t smem_per_block, int parts) {
    PSweep &ps = p.ps;
    const int bs = p.bs, bs2 = bs * bs, vs = ps_vec_stride(bs);
    const int64_t n = p.n;
    const bool timing = std::getenv("BILUK_PLAN_TIMING") != nullptr;
    auto last = std::chrono::steady_clock::now();
    auto tick = [&](const char *what) {   // diagnostics: phase times (BILUK_PLAN_TIMING)
        const auto now = std::chrono::steady_clock::now();
        if (timing) std::fprintf(stderr, "[plan]   %s %.3f s\n", what, std::chrono::duration<double>(now - last).count());
        last = now;
    };
    // ---- choose the partition ---------------------------------------------------
    // ILU(0) on a structured grid: (y, z) columns.  With fill (k >= 1) a row
    // also depends on rows of the next column over in y (fill entries such as
    // (x+1, y-1)), so column parts wait on each other level after level;
    // contiguous row ranges keep every dependency flowing from a part to
    // later parts and measured 1.5x faster.  Anything that is
    // not a grid: contiguous.  BILUK_PARTITION=columns|contiguous overrides.
    // P: every SM for large systems, else the cost model's choice.
    int64_t g[3] = {0, 0, 0};
    const bool is_grid = detect_grid(p, g);
    bool grid = is_grid && p.k == 0;
    if (const char *env = std::getenv("BILUK_PARTITION")) {
        if (std::string(env) == "contiguous") grid = false;
        if (std::string(env) == "columns") grid = is_grid;
    }
    int P = parts;
    if (const char *env = std::getenv("BILUK_PARTS")) P = std::atoi(env);
    Partition pt;
    auto make = [&](int cand, Partition &out) {
        cand = int(std::max<int64_t>(1, std::min<int64_t>(cand, std::max<int64_t>(1, n))));
        if (grid)
            partition_columns(p, cand, g, out);
        else
            partition_contiguous(p, cand, out);
        partition_finish(out);
    };
    ps.est_us = 0;
    if (P > 0 || n >= int64_t(num_sms) * 4096) {
        make(P > 0 ? std::min(P, num_sms) : num_sms, pt);
    } else {
        double best = 1e300;
        for (int cand = num_sms; cand >= 1; cand /= 2) {
            Partition c;
            make(cand, c);
            const double e = psweep_estimate_us(p, c);
            if (e < best * 0.97) {
                best = e;
                pt = std::move(c);
            }
        }
        ps.est_us = best;
    }
    P = pt.P;
    ps.P = P;
    ps.partition = pt.kind;
    for (int d = 0; d < 3; ++d) ps.grid[d] = pt.grid[d];
    ps.split[0] = pt.split[0];
    ps.split[1] = pt.split[1];
    // ---- shared-memory budget of one CTA ---------------------------------------
    ps.nthreads = 128;   // rows per record = threads of a compute group
    // vector ring rows: two levels of a part suffice for ILU(0) / ILU(1)
    // (dependencies one level back; the smaller ring leaves the records more
    // room: 128^3 ILU(0) 515 -> 511 us, ILU(1) 1500 -> 1487 us); ILU(2)+ reach
    // further back (256 rows measured 34 us slower there)
    ps.ring = (bs > 4 || p.k <= 1) ? 256 : 512;
    const int64_t vring = align128(int64_t(ps.ring + 2) * vs * 8);
    ps.xval_ring = 0;   // fetched values live in each record's footprint
    const int64_t budget = int64_t(smem_per_block) - 2048;   // static shared + barriers
    ps.data_ring = ((budget - vring - ps.xval_ring) / 1024) * 1024;
    if (ps.data_ring < 16 * 1024) return fail(BILUK_EUNSUPPORTED, "not enough shared memory for the sweep");
    ps.rec_cap = std::min<int64_t>(ps.data_ring / 4, 48 * 1024);
    ps.glob_cap = ps_glob_cap(bs);

    ps.posL.assign(n, -1);
    ps.posU.assign(n, -1);
    std::vector<std::vector<int32_t>> ordL(P), ordU(P);
    parallel_parts(P, [&](int c) {
        part_order(p.lev_L, pt.rows[c], ordL[c]);
        part_order(p.lev_U, pt.rows[c], ordU[c]);
        for (size_t q = 0; q < ordL[c].size(); ++q) ps.posL[ordL[c][q]] = int32_t(pt.base[c] + q);
        for (size_t q = 0; q < ordU[c].size(); ++q) ps.posU[ordU[c][q]] = int32_t(pt.base[c] + q);
    });

    // the records of every part, built independently (threads), then
    // concatenated: offsets inside a part are relative until the merge
    tick("partition and row orders");
    std::vector<PartRecords> built(P);
    parallel_parts(P, [&](int c) { build_part_records(p, pt, ordL[c], ordU[c], c, built[c]); });
    tick("part records");
    // concatenate: every part's share of the record, index and value-map
    // arrays is known up front, so the parts are copied into place in parallel
    ps.part_rec.assign(P + 1, 0);
    std::vector<int32_t> part_nl(P, 0);   // L records of each part
    std::vector<int64_t> base_rec(P + 1, 0), base_bytes(P + 1, 0), base_idx(P + 1, 0), base_vmap(P + 1, 0);
    ps.rec_total = ps.max_rec = ps.max_glob = ps.nglob_total = 0;
    ps.nlrec_max = 0;
    for (int c = 0; c < P; ++c) {
        const PartRecords &pr = built[c];
        if (pr.rc != BILUK_OK) return fail(pr.rc, pr.msg);
        ps.part_rec[c] = int32_t(base_rec[c]);
        part_nl[c] = pr.nl;
        ps.nlrec_max = std::max<int32_t>(ps.nlrec_max, pr.nl);
        base_rec[c + 1] = base_rec[c] + int64_t(pr.rec.size());
        base_bytes[c + 1] = base_bytes[c] + pr.rec_total;
        base_idx[c + 1] = base_idx[c] + int64_t(pr.idx.size());
        base_vmap[c + 1] = base_vmap[c] + int64_t(pr.vmap.size());
        ps.max_rec = std::max(ps.max_rec, pr.max_rec);
        ps.max_glob = std::max(ps.max_glob, pr.max_glob);
        ps.nglob_total += pr.nglob_total;
    }
    ps.rec_total = base_bytes[P];
    ps.rec.resize(size_t(base_rec[P]));
    ps.idx.resize(size_t(base_idx[P]));
    ps.vmap.resize(size_t(base_vmap[P]));
    parallel_parts(P, [&](int c) {
        PartRecords &pr = built[c];
        PRecInfo *dst = ps.rec.data() + base_rec[c];
        for (size_t r = 0; r < pr.rec.size(); ++r) {
            PRecInfo info = pr.rec[r];
            info.off += uint64_t(base_bytes[c]);
            info.idx_off += uint64_t(base_idx[c]);
            info.vmap_off += base_vmap[c];
            dst[r] = info;
        }
        std::copy(pr.idx.begin(), pr.idx.end(), ps.idx.begin() + base_idx[c]);
        std::copy(pr.vmap.begin(), pr.vmap.end(), ps.vmap.begin() + base_vmap[c]);
        pr = PartRecords();   // free as we go
    });
    tick("merge");
    ps.part_rec[P] = int32_t(ps.rec.size());
    ps.part_rec.insert(ps.part_rec.end(), part_nl.begin(), part_nl.end());   // then P L-record counts
    if (ps.rec.size() >= size_t(INT32_MAX)) return fail(BILUK_EUNSUPPORTED, "too many sweep records");
    // a row is published to the tagged global vector only if some record
    // fetches it (other parts, or rows that left the ring): mark it in iarr
    {
        std::vector<uint8_t> need[2] = {std::vector<uint8_t>(n, 0), std::vector<uint8_t>(n, 0)};
        for (const PRecInfo &ri : ps.rec) {
            const int32_t *gp = ps.idx.data() + ri.idx_off + sizeof(PRecHdr) / 4 + ri.nrows + rec_desc_words(ri.nrows, ri.S);
            for (int t = 0; t < ri.nglob; ++t) need[ri.level & 1][gp[t]] = 1;
        }
        for (const PRecInfo &ri : ps.rec) {
            int32_t *iarr = ps.idx.data() + ri.idx_off + sizeof(PRecHdr) / 4;
            for (int q = 0; q < ri.nrows; ++q)
                if (need[ri.level & 1][ri.pos0 + q]) iarr[q] = int32_t(uint32_t(iarr[q]) | 0x80000000u);
        }
    }
    // fault injection (tests only): the first record that fetches a
    // dependency instead waits on its own first row, which is published after
    // it -- the sweep must time out with BILUK_ETIMEOUT, not hang
    if (const char *env = std::getenv("BILUK_FAULT_GPOS")) {
        if (std::atoi(env) == 1)
            for (const PRecInfo &ri : ps.rec)
                if (ri.nglob > 0) {
                    ps.idx[ri.idx_off + sizeof(PRecHdr) / 4 + ri.nrows + rec_desc_words(ri.nrows, ri.S)] = ri.pos0;
                    break;
                }
    }
    return BILUK_OK;
}

}  // namespace biluk
