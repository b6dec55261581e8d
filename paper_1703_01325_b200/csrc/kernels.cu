// Device kernels of the block ILU(k) path for sm_100a:
//   materialize   A -> A' on the ILU(k) pattern            (factor.py:83-121)
//   factor_level  block IKJ ILU(0), one warp per block row  (factor.py:165-205)
//   split         U'_ij = D_i^-1 U_ij                       (factor.py:230-289)
//   pack_sweep    factors -> level-ordered tile records
//   sweep         persistent sync-free L and U' sweeps      (trisolve.py:121-182)
//   spmv          sliced-ELL BSR SpMV                       (sparse.py:278-301)
#include <cstdint>

#include "biluk_internal.h"
#include "device_util.cuh"
#include "kernels.cuh"

namespace biluk {

using namespace dev;

// ===========================================================================
// materialize: scatter the original blocks into the zeroed P' value array
// ===========================================================================
__global__ void materialize_kernel(const int32_t *__restrict__ a2p, int64_t nnzA, int bs2,
                                   const double *__restrict__ avals, double *__restrict__ pvals) {
    const int64_t total = nnzA * bs2;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t slot = g / bs2;
        const int e = int(g - slot * bs2);
        pvals[int64_t(a2p[slot]) * bs2 + e] = avals[g];
    }
}

// ===========================================================================
// factor one dependency level: warp per block row, the row staged in shared
// memory.  IKJ order of block_ilu0_factorize (factor.py:184-204):
//   for lower slot t (ascending pivot p):  A_ip <- A_ip D_p^-1
//        for every stored U_pj of row p with (i, j) stored:  A_ij -= A_ip U_pj
//   D_i^-1 = inv(A_ii)
// bs == 1 follows the point kernel (factor.py:124-148): division by the
// pivot, |pivot| < 1e-300 is a zero pivot.  U stays unscaled here (the split
// kernel runs after the whole factorization).
// ===========================================================================
template <int BS>
__global__ void factor_level_kernel(const int32_t *__restrict__ rows, int64_t nrows, const int32_t *__restrict__ rp,
                                    const int32_t *__restrict__ ci, const int32_t *__restrict__ diag,
                                    double *__restrict__ pvals, double *__restrict__ dinv, DevStatus *st,
                                    int maxlen) {
    constexpr int BS2 = BS * BS;
    extern __shared__ double fsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gw = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
    if (gw >= nrows) return;
    const int32_t i = rows[gw];
    const int32_t s = rp[i], e = rp[i + 1], d = diag[i];
    const int len = e - s;
    double *W = fsm + size_t(warp) * maxlen * BS2;
    for (int x = lane; x < len * BS2; x += 32) W[x] = pvals[int64_t(s) * BS2 + x];
    __syncwarp();
    for (int t = s; t < d; ++t) {
        const int32_t p = ci[t];
        double *Wt = W + (t - s) * BS2;
        // A_ip <- A_ip D_p^-1  (bs==1: A_ip / U_pp)
        constexpr int NE = (BS2 + 31) / 32;
        double lv[NE];
#pragma unroll
        for (int q = 0; q < NE; ++q) {
            const int el = lane + 32 * q;
            lv[q] = 0.0;
            if (el < BS2) {
                const int r = el % BS, c = el / BS;
                if (BS == 1) {
                    lv[q] = Wt[0] / pvals[int64_t(diag[p])];
                } else {
                    const double *Dp = dinv + int64_t(p) * BS2;
#pragma unroll
                    for (int m = 0; m < BS; ++m) lv[q] += Wt[m * BS + r] * Dp[c * BS + m];
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NE; ++q)
            if (lane + 32 * q < BS2) Wt[lane + 32 * q] = lv[q];
        __syncwarp();
        // A_ij -= A_ip U_pj for the stored (i, j), j > p
        const int32_t us = diag[p] + 1, ue = rp[p + 1];
        const int tasks = (ue - us) * BS2;
        for (int task = lane; task < tasks; task += 32) {
            const int u = us + task / BS2, el = task % BS2;
            const int32_t j = ci[u];
            int lo = t + 1 - s, hi = len;   // j > p: search right of slot t
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (ci[s + mid] < j) lo = mid + 1; else hi = mid;
            }
            if (lo < len && ci[s + lo] == j) {
                const int r = el % BS, c = el / BS;
                const double *U = pvals + int64_t(u) * BS2;
                double acc = 0.0;
#pragma unroll
                for (int m = 0; m < BS; ++m) acc += Wt[m * BS + r] * U[c * BS + m];
                W[lo * BS2 + el] -= acc;
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        const double *Dii = W + (d - s) * BS2;
        bool ok;
        if (BS == 1) {
            ok = fabs(Dii[0]) >= 1e-300;
            if (ok) dinv[i] = 1.0 / Dii[0];
        } else {
            double inv[BS2];
            ok = block_invert<BS>(Dii, inv);
#pragma unroll
            for (int x = 0; x < BS2; ++x) dinv[int64_t(i) * BS2 + x] = ok ? inv[x] : 0.0;
        }
        if (!ok) {
            atomicExch(&st->fstatus, BS == 1 ? BILUK_EZEROPIVOT : BILUK_ESINGULAR);
            atomicMin(&st->ferr_row, (long long)i);
        }
    }
    __syncwarp();
    for (int x = lane; x < len * BS2; x += 32) pvals[int64_t(s) * BS2 + x] = W[x];
}

// ===========================================================================
// split: U'_ij = D_i^-1 U_ij in place on the strictly-upper slots
// (factor.py:266-268); one thread per block row.
// ===========================================================================
template <int BS>
__global__ void split_kernel(int64_t n, const int32_t *__restrict__ rp, const int32_t *__restrict__ diag,
                             const double *__restrict__ dinv, double *__restrict__ pvals) {
    constexpr int BS2 = BS * BS;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        double D[BS2];
#pragma unroll
        for (int x = 0; x < BS2; ++x) D[x] = dinv[i * BS2 + x];
        for (int32_t u = diag[i] + 1; u < rp[i + 1]; ++u) {
            double *U = pvals + int64_t(u) * BS2;
            double in[BS2];
#pragma unroll
            for (int x = 0; x < BS2; ++x) in[x] = U[x];
#pragma unroll
            for (int c = 0; c < BS; ++c)
#pragma unroll
                for (int r = 0; r < BS; ++r) {
                    double acc = 0.0;
#pragma unroll
                    for (int m = 0; m < BS; ++m) acc += D[m * BS + r] * in[c * BS + m];
                    U[c * BS + r] = acc;
                }
        }
    }
}

// ===========================================================================
// pack one sweep's tile records from the factored P' values (thread per
// tile lane).  L tiles take the row's strictly-lower slots, U' tiles the
// strictly-upper ones plus D^-1 of the row; padding rows/slots get -1 / 0.
// ===========================================================================
template <int BS>
__global__ void pack_sweep_kernel(int64_t ntiles, const TileMeta *__restrict__ meta, const int32_t *__restrict__ trows,
                                  unsigned char *__restrict__ rec, bool upper, const int32_t *__restrict__ rp,
                                  const int32_t *__restrict__ ci, const int32_t *__restrict__ diag,
                                  const double *__restrict__ pvals, const double *__restrict__ dinv,
                                  const int32_t *__restrict__ pos_dep, const int32_t *__restrict__ pos_l) {
    constexpr int R = rows_per_tile(BS);
    constexpr int BS2 = BS * BS;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < ntiles * R; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = g / R;
        const int lane = int(g - t * R);
        const TileMeta m = meta[t];
        const int S = m.nslot;
        unsigned char *r0 = rec + int64_t(m.off128) * 128;
        const int32_t row = trows[g];
        reinterpret_cast<int32_t *>(r0)[lane] = row;
        if (upper) reinterpret_cast<int32_t *>(r0 + 128)[lane] = row >= 0 ? pos_l[row] : -1;
        int32_t base = 0, cnt = 0;
        if (row >= 0) {
            base = upper ? diag[row] + 1 : rp[row];
            cnt = upper ? rp[row + 1] - diag[row] - 1 : diag[row] - rp[row];
        }
        int32_t *cols = reinterpret_cast<int32_t *>(r0 + rec_hdr_bytes(upper));
        double *vals = reinterpret_cast<double *>(r0 + rec_vals_off(BS, S, upper));
        for (int s = 0; s < S; ++s) {
            const bool live = s < cnt;
            cols[s * R + lane] = live ? pos_dep[ci[base + s]] : -1;
            const double *src = pvals + int64_t(base + s) * BS2;
            for (int x = 0; x < BS2; ++x) vals[(int64_t(s) * BS2 + x) * R + lane] = live ? src[x] : 0.0;
        }
        if (upper) {
            double *dv = reinterpret_cast<double *>(r0 + rec_dinv_off(BS, S));
            for (int x = 0; x < BS2; ++x) dv[x * R + lane] = row >= 0 ? dinv[int64_t(row) * BS2 + x] : 0.0;
        }
    }
}

// ===========================================================================
// pack the sliced-ELL copy of A used by SpMV (natural row order)
// ===========================================================================
template <int BS>
__global__ void pack_ell_kernel(int64_t n, int64_t ntiles, const TileMeta *__restrict__ meta, unsigned char *__restrict__ rec,
                                const int32_t *__restrict__ arp, const int32_t *__restrict__ aci,
                                const double *__restrict__ avals) {
    constexpr int R = rows_per_tile(BS);
    constexpr int BS2 = BS * BS;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < ntiles * R; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = g / R;
        const int lane = int(g - t * R);
        const TileMeta m = meta[t];
        const int S = m.nslot;
        unsigned char *r0 = rec + int64_t(m.off128) * 128;
        const int64_t row = g;
        int32_t base = 0, cnt = 0;
        if (row < n) {
            base = arp[row];
            cnt = arp[row + 1] - base;
        }
        int32_t *cols = reinterpret_cast<int32_t *>(r0);
        double *vals = reinterpret_cast<double *>(r0 + ell_vals_off(BS, S));
        for (int s = 0; s < S; ++s) {
            const bool live = s < cnt;
            cols[s * R + lane] = live ? aci[base + s] : -1;
            for (int x = 0; x < BS2; ++x)
                vals[(int64_t(s) * BS2 + x) * R + lane] = live ? avals[int64_t(base + s) * BS2 + x] : 0.0;
        }
    }
}

// ===========================================================================
// The sweep: ONE persistent kernel for L y = b and U' x = D^-1 y.
//
// Tiles are dealt statically: warp w of W owns tiles w, w+W, w+2W, ... of the
// sequence [L tiles in level order | U' tiles in level order].  Every
// dependency of a tile lives in a strictly earlier tile, all W warps are
// co-resident (cooperative launch), so the smallest unfinished tile can
// always make progress: no deadlock.  Each warp keeps `stages` tile records
// in flight in shared memory (one bulk async copy each, issued as soon as a
// buffer frees up), so matrix streaming is decoupled from the dependency
// chain; only the vector values travel along it.  A lane owns one block row:
//   L :  y_i = b_i - sum_j L_ij y_j
//   U':  x_i = D_i^-1 y_i - sum_j U'_ij x_j
// Dependencies are polled directly on the parity-tagged rows (see tag_row()),
// ONE component per dependency until it is published, then the rest.  To keep
// the polls from flooding L2, a warp first waits (one load per warp, with
// back-off) until every level <= its own level - gap is complete: per-level
// tile counters advance a `prefix` of completed levels (a progress hint only;
// correctness rests on the value tags).
// ===========================================================================
__device__ __forceinline__ void fence_sc() { asm volatile("fence.sc.gpu;" ::: "memory"); }

// Wait budget, checked every 256 spins against the SM cycle counter (cheap,
// unlike %globaltimer); budget = timeout_ns * 2 cycles (>= timeout_ns at <= 2 GHz).
__device__ __forceinline__ bool timed_out(uint64_t &t0, uint32_t &spins, const SweepArgs &a) {
    ++spins;
    if (spins == 1) {
        t0 = uint64_t(clock64());
    } else if ((spins & 255u) == 0) {
        if (uint64_t(clock64()) - t0 > 2 * a.timeout_ns || ld_relaxed_s32(&a.st->status) != 0) {
            atomicCAS(&a.st->status, 0, int(BILUK_ETIMEOUT));
            return true;
        }
    }
    return false;
}

// Wait for NE published values: entry e has its BS components at
// p[e] + q * stride.  Every poll round issues ALL pending loads before
// looking at any of them, so one round costs one L2 round trip however many
// dependencies a row has (checking each value right after its own load would
// serialise one round trip per dependency).  Values come back exact (untag_row).
template <int BS, int NE>
__device__ __forceinline__ void wait_values(const double *__restrict__ base, const double *__restrict__ last_base,
                                            const int (&pos)[NE], double (&xv)[NE][BS], uint32_t pend, uint32_t par,
                                            const SweepArgs &a) {
    // entry e < NE-1 is the row at position pos[e] of base, the last entry of last_base;
    // a row is tag_stride(BS) contiguous doubles
    uint64_t t0 = 0;
    uint32_t spins = 0;
#pragma unroll
    for (int e = 0; e < NE; ++e)
#pragma unroll
        for (int q = 0; q < BS; ++q) xv[e][q] = 0.0;   // entries never polled contribute zero
    // the LSB words of the entries (their values land in xv directly)
    double lw[NE];
    while (pend) {
        // issue every pending load, then look at them (one round trip per round)
#pragma unroll
        for (int e = 0; e < NE; ++e)
            if (pend & (1u << e))
                ld_tagged_split<BS>((e == NE - 1 ? last_base : base) + int64_t(pos[e]) * tag_stride(BS), xv[e], lw[e]);
        uint32_t still = 0;
#pragma unroll
        for (int e = 0; e < NE; ++e)
            if (pend & (1u << e)) {
                uint32_t ok = tag_of(lw[e]) == par;
#pragma unroll
                for (int c = 0; c < BS; ++c) ok &= (tag_of(xv[e][c]) == par);
                if (ok)
                    untag_split<BS>(xv[e], lw[e]);
                else
                    still |= 1u << e;
            }
        pend &= still;
        if (!pend) break;
        if (timed_out(t0, spins, a)) break;
        if (a.fine_sleep_ns) __nanosleep(a.fine_sleep_ns);
    }
}

// the finisher of a level tries to advance the completed-level prefix
__device__ __forceinline__ void advance_prefix(uint32_t l, const SweepArgs &a) {
    while (true) {
        if (ld_relaxed_u32(&a.st->prefix) != l - 1) return;
        if (atomicCAS(&a.st->prefix, l - 1, l) != l - 1) return;
        fence_sc();
        ++l;
        if (int(l) > a.nlev_total) return;
        if (ld_relaxed_u32(a.lvl_cnt + l) != a.lvl_tiles[l]) return;
    }
}

// One lane's block row of a tile: poll its dependencies (CH per round) and
// accumulate  acc -= sum_s B_s x_s  (U' rows first set acc = D^-1 y_i).
// The first CHR slots' blocks and D^-1 are staged in registers BEFORE the
// poll, so once the dependencies arrive only register FMAs remain; padding
// slots hold zero blocks and zero x, so no per-lane guards are needed.
template <int BS, int CH, int CHR>
__device__ __forceinline__ void row_solve(const SweepArgs &a, const unsigned char *rec, int S, bool up, int lane,
                                          uint32_t par, double (&acc)[BS], uint64_t &tr_deps, long long &cyc_deps) {
    constexpr int R = rows_per_tile(BS);
    constexpr int BS2 = BS * BS;
    constexpr bool STAGE = BS <= 4;
    const int *cols = reinterpret_cast<const int *>(rec + rec_hdr_bytes(up));
    const double *vals = reinterpret_cast<const double *>(rec + rec_vals_off(BS, S, up));
    const double *dep = up ? a.x_t : a.y_t;
    double vr[CHR > 0 ? CHR : 1][BS2];
    double dr[STAGE ? BS2 : 1];
    const double *dv = reinterpret_cast<const double *>(rec + rec_dinv_off(BS, S)) + lane;
#pragma unroll
    for (int c = 0; c < CHR; ++c)
#pragma unroll
        for (int x = 0; x < BS2; ++x) vr[c][x] = c < S ? vals[(size_t(c) * BS2 + x) * R + lane] : 0.0;
    if (STAGE && up) {
#pragma unroll
        for (int x = 0; x < (STAGE ? BS2 : 1); ++x) dr[x] = dv[x * R];
    }
    for (int s0 = 0; s0 < S || (up && s0 == 0); s0 += CH) {
        // entries 0..CH-1: dependencies of this chunk; entry CH: the row's own
        // y_i (U' tiles, first chunk), polled in the same round
        int pp[CH + 1];
        double xv[CH + 1][BS];
        uint32_t pend = 0;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int j = (s0 + c < S) ? cols[(s0 + c) * R + lane] : -1;
            pp[c] = j >= 0 ? j : 0;
            if (j >= 0) pend |= 1u << c;
        }
        pp[CH] = up ? reinterpret_cast<const int *>(rec + 128)[lane] : 0;
        if (up && s0 == 0) pend |= 1u << CH;
        wait_values<BS, CH + 1>(dep, a.y_t, pp, xv, pend, par, a);
        if (a.trace && lane == 0 && s0 == 0) {
            tr_deps = globaltimer();
            cyc_deps = clock64();
        }
        if (up && s0 == 0) {
#pragma unroll
            for (int r = 0; r < BS; ++r) {
                double z = (STAGE ? dr[r % (STAGE ? BS2 : 1)] : dv[r * R]) * xv[CH][0];
#pragma unroll
                for (int c = 1; c < BS; ++c)
                    z = fma(STAGE ? dr[(c * BS + r) % (STAGE ? BS2 : 1)] : dv[(c * BS + r) * R], xv[CH][c], z);
                acc[r] = z;
            }
        }
        // register-staged slots (first chunk): all chains in parallel, then a
        // pairwise tree into acc; remaining slots: warp-uniform shared-memory loop
        if (s0 == 0 && CHR > 0) {
            double pr[CHR > 0 ? CHR : 1][BS];
#pragma unroll
            for (int c = 0; c < CHR; ++c)
#pragma unroll
                for (int r = 0; r < BS; ++r) {
                    double p = vr[c][r] * xv[c][0];
#pragma unroll
                    for (int q = 1; q < BS; ++q) p = fma(vr[c][q * BS + r], xv[c][q], p);
                    pr[c][r] = p;
                }
#pragma unroll
            for (int w = 1; w < CHR; w <<= 1)
#pragma unroll
                for (int c = 0; c + w < CHR; c += 2 * w)
#pragma unroll
                    for (int r = 0; r < BS; ++r) pr[c][r] += pr[c + w][r];
#pragma unroll
            for (int r = 0; r < BS; ++r) acc[r] -= pr[0][r];
        }
        const int cstart = s0 == 0 ? CHR : 0;
        if (s0 + cstart < S)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (c >= cstart && s0 + c < S) {
                    const double *v = vals + size_t(s0 + c) * BS2 * R + lane;
                    double pr[BS];
#pragma unroll
                    for (int r = 0; r < BS; ++r) pr[r] = v[r * R] * xv[c][0];
#pragma unroll
                    for (int q = 1; q < BS; ++q)
#pragma unroll
                        for (int r = 0; r < BS; ++r) pr[r] = fma(v[(q * BS + r) * R], xv[c][q], pr[r]);
#pragma unroll
                    for (int r = 0; r < BS; ++r) acc[r] -= pr[r];
                }
            }
    }
}

template <int BS>
__global__ void __launch_bounds__(256, 1) sweep_kernel(const SweepArgs a) {
    constexpr int R = rows_per_tile(BS);
    constexpr int BS2 = BS * BS;
    constexpr int CH = BS <= 4 ? 8 : (BS <= 6 ? 6 : 4);
    // register-staged slots per row: ~27 doubles of matrix values (none for bs > 4)
    constexpr int CHR = BS > 4 ? 0 : (BS == 4 ? 1 : ((27 / BS2) < CH ? (27 / BS2) : CH));
    constexpr int CHS = BS <= 3 ? 4 : (BS <= 4 ? 2 : 1);   // narrow-tile poll width
    constexpr int CHS_R = CHR < CHS ? CHR : CHS;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int last_cta;
    __shared__ uint32_t cta_prefix;
    if (a.skip_flag && ld_relaxed_s32(a.skip_flag) != 0) return;
    if (threadIdx.x == 0) cta_prefix = 0;
    __syncthreads();
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * a.stages;
    unsigned char *stage0 = smem + align128(int64_t(nw) * a.stages * 8) + size_t(warp) * a.stages * a.stage_bytes;
    const uint32_t par = ld_relaxed_u32(&a.st->epoch) & 1u;
    const int64_t W = int64_t(gridDim.x) * nw;
    const int64_t w0 = int64_t(blockIdx.x) * nw + warp;
    const int64_t T = a.nl + a.nu;
    const uint64_t pol = policy_evict_first();

    auto issue = [&](int64_t t, int s) {
        const bool up = t >= a.nl;
        const TileMeta m = up ? a.meta_u[t - a.nl] : a.meta_l[t];
        const unsigned char *src = (up ? a.rec_u : a.rec_l) + int64_t(m.off128) * 128;
        const uint32_t bytes = uint32_t(rec_bytes(BS, m.nslot, up));
        mbar_expect_tx(bars + s, bytes);
        bulk_g2s(stage0 + size_t(s) * a.stage_bytes, src, bytes, bars + s, pol);
    };

    if (lane == 0) {
        for (int s = 0; s < a.stages; ++s) mbar_init(bars + s, 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0)
        for (int s = 0; s < a.stages; ++s)
            if (w0 + s * W < T) issue(w0 + s * W, s);

    int64_t k = 0;
    for (int64_t t = w0; t < T; t += W, ++k) {
        const int s = int(k % a.stages);
        const uint32_t ph = uint32_t(k / a.stages) & 1u;
        const bool up = t >= a.nl;
        const TileMeta m = up ? a.meta_u[t - a.nl] : a.meta_l[t];
        const int S = m.nslot;
        const uint32_t lvl = uint32_t(up ? a.nlev_l + m.level : m.level);
        mbar_wait(bars + s, ph);
        const unsigned char *rec = stage0 + size_t(s) * a.stage_bytes;
        const int row = lane < R ? reinterpret_cast<const int *>(rec)[lane] : -1;
        double acc[BS];
        if (row >= 0 && !up) {
#pragma unroll
            for (int r = 0; r < BS; ++r) acc[r] = __ldg(a.b + int64_t(row) * BS + r);
        }
        uint64_t tr0 = 0;
        if (a.trace && lane == 0) tr0 = globaltimer();
        // coarse wait: one lane per warp; the CTA shares the last prefix value
        // it saw (shared memory) so the global word is read at most by a few
        // warps, and the back-off grows with the distance to the target level
        if (lane == 0 && a.gap > 0 && int(lvl) - a.gap > 0) {
            const int target = int(lvl) - a.gap;
            uint64_t t0 = 0;
            uint32_t spins = 0;
            while (int(*reinterpret_cast<volatile uint32_t *>(&cta_prefix)) < target) {
                const int p = int(ld_relaxed_u32(&a.st->prefix));
                atomicMax(&cta_prefix, uint32_t(p));
                if (p >= target) break;
                if (timed_out(t0, spins, a)) break;
                const int d = target - p;
                __nanosleep(uint32_t(min(a.coarse_sleep_ns * d, 4000)));
            }
        }
        // cheap wait: one lane polls ONE dependency of the previous level (one
        // 8-byte load, back-off) so that warps far ahead of the frontier do
        // not flood their SM's load pipeline with full-warp polls
        const int probe = a.probe == 1 ? m.probe[0] : (a.probe == 2 ? m.probe[1] : -1);
        if (lane == 0 && probe != -1) {
            const double *pv = probe >= 0 ? (up ? a.x_t : a.y_t) + int64_t(probe) * tag_stride(BS) + BS
                                          : a.y_t + int64_t(-probe - 2) * tag_stride(BS) + BS;
            uint64_t t0 = 0;
            uint32_t spins = 0;
            while (tag_of(ld_relaxed(pv)) != par) {
                if (timed_out(t0, spins, a)) break;
                if (a.probe_sleep_ns) __nanosleep(a.probe_sleep_ns);
            }
        }
        __syncwarp();
        uint64_t tr1 = 0, tr_deps = 0;
        long long cyc_deps = 0, cyc_fma = 0, cyc_st = 0;
        if (a.trace && lane == 0) tr1 = globaltimer();
        if (row >= 0) {
            // narrow tiles (<= CHS dependency slots, e.g. every ILU(0) row) use a
            // poll of CHS entries; wider ones the general CH-wide chunked poll
            if (S <= CHS)
                row_solve<BS, CHS, CHS_R>(a, rec, S, up, lane, par, acc, tr_deps, cyc_deps);
            else
                row_solve<BS, CH, CHR>(a, rec, S, up, lane, par, acc, tr_deps, cyc_deps);
            if (a.trace && lane == 0) cyc_fma = clock64();
            // publish the row at its own position: one (or two) vector stores,
            // coalesced across the warp's consecutive positions
            double *dst = (up ? a.x_t : a.y_t) + ((up ? t - a.nl : t) * R + lane) * tag_stride(BS);
            st_tagged<BS>(dst, acc, par);
            if (up && a.out) {
#pragma unroll
                for (int r = 0; r < BS; ++r) a.out[int64_t(row) * BS + r] = acc[r];
            }
            if (a.trace && lane == 0) cyc_st = clock64();
        }
        __syncwarp();
        if (lane == 0) {
            if (a.trace) {
                const long long cyc_done = clock64();
                const unsigned long long packed =
                    (unsigned long long)(cyc_fma - cyc_deps) | ((unsigned long long)(cyc_st - cyc_deps) << 21) |
                    ((unsigned long long)(cyc_done - cyc_deps) << 42);
                ulonglong4 rec4 = make_ulonglong4(tr0, tr1, globaltimer(), a.trace_mode == 2 ? packed : tr_deps);
                reinterpret_cast<ulonglong4 *>(a.trace)[t] = rec4;
            }
            // progress accounting (a hint only): count the tile, advance the
            // completed-level prefix when this tile completes its level
            if (a.gap > 0 && atomicAdd(a.lvl_cnt + lvl, 1u) + 1 == a.lvl_tiles[lvl]) {
                fence_sc();
                advance_prefix(lvl, a);
            }
            if (t + int64_t(a.stages) * W < T) {
                fence_proxy_async();
                issue(t + int64_t(a.stages) * W, s);
            }
        }
    }
    // the last CTA to finish advances the epoch (every CTA read it at entry)
    // and resets the progress counters for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last_cta = atomicAdd(&a.st->done_ctas, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last_cta) {
        __threadfence();
        for (int l = threadIdx.x; l <= a.nlev_total + 1; l += blockDim.x) a.lvl_cnt[l] = 0;
        __syncthreads();
        if (threadIdx.x == 0) {
            a.st->prefix = 0;
            a.st->done_ctas = 0;
            __threadfence();
            atomicAdd(&a.st->epoch, 1u);
        }
    }
}

// ===========================================================================
// SpMV y = A x on the sliced-ELL copy of A: warp per tile, lane per block row
// ===========================================================================
template <int BS>
__global__ void __launch_bounds__(256) spmv_kernel(int64_t n, int64_t ntiles, const TileMeta *__restrict__ meta,
                                                   const unsigned char *__restrict__ rec, const double *__restrict__ x,
                                                   double *__restrict__ y, const int *skip_flag) {
    constexpr int R = rows_per_tile(BS);
    constexpr int BS2 = BS * BS;
    if (skip_flag && ld_relaxed_s32(skip_flag) != 0) return;
    const int lane = threadIdx.x & 31;
    const int64_t W = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t t = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles; t += W) {
        const TileMeta m = meta[t];
        const int64_t row = t * R + lane;
        if (lane >= R || row >= n) continue;
        const unsigned char *r0 = rec + int64_t(m.off128) * 128;
        const int *cols = reinterpret_cast<const int *>(r0);
        const double *vals = reinterpret_cast<const double *>(r0 + ell_vals_off(BS, m.nslot));
        double acc[BS];
#pragma unroll
        for (int r = 0; r < BS; ++r) acc[r] = 0.0;
#pragma unroll 2
        for (int s = 0; s < m.nslot; ++s) {
            const int j = __ldg(cols + s * R + lane);
            if (j < 0) continue;
            double xv[BS];
#pragma unroll
            for (int q = 0; q < BS; ++q) xv[q] = __ldg(x + int64_t(j) * BS + q);
            const double *v = vals + size_t(s) * BS2 * R + lane;
#pragma unroll
            for (int q = 0; q < BS; ++q)
#pragma unroll
                for (int r = 0; r < BS; ++r) acc[r] = fma(__ldg(v + (q * BS + r) * R), xv[q], acc[r]);
        }
#pragma unroll
        for (int r = 0; r < BS; ++r) y[row * BS + r] = acc[r];
    }
}

// ===========================================================================
// host-side launchers (templated dispatch on the block size)
// ===========================================================================
#define BILUK_BS_DISPATCH(bs, F)  \
    switch (bs) {                 \
        case 1: F(1); break;      \
        case 2: F(2); break;      \
        case 3: F(3); break;      \
        case 4: F(4); break;      \
        case 5: F(5); break;      \
        case 6: F(6); break;      \
        case 7: F(7); break;      \
        case 8: F(8); break;      \
        default: return cudaErrorInvalidValue; \
    }

static int grid_for(int64_t work, int threads, int num_sms) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = int64_t(num_sms) * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return int(g);
}

cudaError_t launch_materialize(const Plan &p, const double *avals, cudaStream_t s) {
    const int bs2 = p.bs * p.bs;
    double *pv = reinterpret_cast<double *>(p.ws + p.off.pvals);
    cudaError_t e = cudaMemsetAsync(pv, 0, size_t(p.nnzP) * bs2 * 8, s);
    if (e != cudaSuccess) return e;
    if (p.nnzA == 0) return cudaSuccess;
    materialize_kernel<<<grid_for(p.nnzA * bs2, 256, p.num_sms), 256, 0, s>>>(
        reinterpret_cast<const int32_t *>(p.ws + p.off.a2p), p.nnzA, bs2, avals, pv);
    return cudaGetLastError();
}

cudaError_t launch_factor(const Plan &p, cudaStream_t s) {
    const int warps = 4;
    const size_t smem = size_t(warps) * p.max_row_len * p.bs * p.bs * 8;
    const int32_t *rows = reinterpret_cast<const int32_t *>(p.ws + p.off.forder);
    const int32_t *rp = reinterpret_cast<const int32_t *>(p.ws + p.off.p_rp);
    const int32_t *ci = reinterpret_cast<const int32_t *>(p.ws + p.off.p_ci);
    const int32_t *dg = reinterpret_cast<const int32_t *>(p.ws + p.off.p_diag);
    double *pv = reinterpret_cast<double *>(p.ws + p.off.pvals);
    double *dv = reinterpret_cast<double *>(p.ws + p.off.dinv);
    DevStatus *st = reinterpret_cast<DevStatus *>(p.ws + p.off.status);
#define FACTOR_LAUNCH(BS)                                                                                    \
    {                                                                                                        \
        auto kern = factor_level_kernel<BS>;                                                                 \
        if (smem > 48 * 1024) {                                                                              \
            cudaError_t e0 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
            if (e0 != cudaSuccess) return e0;                                                                \
        }                                                                                                    \
        for (int l = 1; l <= p.nlev_L; ++l) {                                                                \
            const int64_t b = p.fptr[l - 1], cnt = p.fptr[l] - b;                                            \
            if (cnt == 0) continue;                                                                          \
            const int64_t grid = (cnt + warps - 1) / warps;                                                  \
            kern<<<unsigned(grid), warps * 32, smem, s>>>(rows + b, cnt, rp, ci, dg, pv, dv, st, p.max_row_len); \
        }                                                                                                    \
    }
    BILUK_BS_DISPATCH(p.bs, FACTOR_LAUNCH)
#undef FACTOR_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_split(const Plan &p, cudaStream_t s) {
    const int32_t *rp = reinterpret_cast<const int32_t *>(p.ws + p.off.p_rp);
    const int32_t *dg = reinterpret_cast<const int32_t *>(p.ws + p.off.p_diag);
    double *pv = reinterpret_cast<double *>(p.ws + p.off.pvals);
    const double *dv = reinterpret_cast<const double *>(p.ws + p.off.dinv);
#define SPLIT_LAUNCH(BS) split_kernel<BS><<<grid_for(p.n, 128, p.num_sms), 128, 0, s>>>(p.n, rp, dg, dv, pv);
    BILUK_BS_DISPATCH(p.bs, SPLIT_LAUNCH)
#undef SPLIT_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_pack(const Plan &p, cudaStream_t s) {
    const int R = rows_per_tile(p.bs);
    const int32_t *rp = reinterpret_cast<const int32_t *>(p.ws + p.off.p_rp);
    const int32_t *ci = reinterpret_cast<const int32_t *>(p.ws + p.off.p_ci);
    const int32_t *dg = reinterpret_cast<const int32_t *>(p.ws + p.off.p_diag);
    const double *pv = reinterpret_cast<const double *>(p.ws + p.off.pvals);
    const double *dv = reinterpret_cast<const double *>(p.ws + p.off.dinv);
    const int32_t *pl = reinterpret_cast<const int32_t *>(p.ws + p.off.pos_l);
    const int32_t *pu = reinterpret_cast<const int32_t *>(p.ws + p.off.pos_u);
#define PACK_LAUNCH(BS)                                                                                        \
    {                                                                                                          \
        if (p.sl.ntiles)                                                                                       \
            pack_sweep_kernel<BS><<<grid_for(p.sl.ntiles * R, 128, p.num_sms), 128, 0, s>>>(                   \
                p.sl.ntiles, reinterpret_cast<const TileMeta *>(p.ws + p.off.sl_meta),                         \
                reinterpret_cast<const int32_t *>(p.ws + p.off.sl_rows), p.ws + p.off.sl_rec, false, rp, ci, dg, pv, dv, \
                pl, pl);                                                                                       \
        if (p.su.ntiles)                                                                                       \
            pack_sweep_kernel<BS><<<grid_for(p.su.ntiles * R, 128, p.num_sms), 128, 0, s>>>(                   \
                p.su.ntiles, reinterpret_cast<const TileMeta *>(p.ws + p.off.su_meta),                         \
                reinterpret_cast<const int32_t *>(p.ws + p.off.su_rows), p.ws + p.off.su_rec, true, rp, ci, dg, pv, dv, \
                pu, pl);                                                                                       \
    }
    BILUK_BS_DISPATCH(p.bs, PACK_LAUNCH)
#undef PACK_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_pack_ell(const Op &o, const double *avals, cudaStream_t s) {
    if (o.ntiles == 0) return cudaSuccess;
    const int R = rows_per_tile(o.bs);
    const int32_t *arp = reinterpret_cast<const int32_t *>(o.ws + o.off.rp);
    const int32_t *aci = reinterpret_cast<const int32_t *>(o.ws + o.off.ci);
    const TileMeta *meta = reinterpret_cast<const TileMeta *>(o.ws + o.off.meta);
#define PACKE_LAUNCH(BS)                                                                                   \
    pack_ell_kernel<BS><<<grid_for(o.ntiles * R, 128, o.num_sms), 128, 0, s>>>(o.n, o.ntiles, meta, o.ws + o.off.rec, \
                                                                             arp, aci, avals);
    BILUK_BS_DISPATCH(o.bs, PACKE_LAUNCH)
#undef PACKE_LAUNCH
    return cudaGetLastError();
}

static int launch_warps(const Plan &p) {
    return (p.tune.warps > 0 && p.tune.warps < p.sweep_warps) ? p.tune.warps : p.sweep_warps;
}

size_t sweep_smem_bytes(const Plan &p) {
    const int w = launch_warps(p);
    return size_t(align128(int64_t(w) * p.sweep_stages * 8)) + size_t(w) * p.sweep_stages * size_t(p.stage_bytes);
}

cudaError_t launch_sweep(const Plan &p, const SweepArgs &a, cudaStream_t s) {
    const size_t smem = sweep_smem_bytes(p);
    dim3 grid(p.sweep_ctas), block(launch_warps(p) * 32);
#define SWEEP_LAUNCH(BS)                                                                                   \
    {                                                                                                      \
        auto kern = sweep_kernel<BS>;                                                                      \
        cudaError_t e0 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        if (e0 != cudaSuccess) return e0;                                                                  \
        void *args[] = {const_cast<SweepArgs *>(&a)};                                                      \
        e0 = cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kern), grid, block, args, smem, s); \
        if (e0 != cudaSuccess) return e0;                                                                  \
    }
    BILUK_BS_DISPATCH(p.bs, SWEEP_LAUNCH)
#undef SWEEP_LAUNCH
    return cudaGetLastError();
}

cudaError_t sweep_occupancy(const Plan &p, int *blocks_per_sm) {
    const size_t smem = sweep_smem_bytes(p);
#define OCC(BS)                                                                                                   \
    {                                                                                                             \
        auto kern = sweep_kernel<BS>;                                                                             \
        cudaError_t e0 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));      \
        if (e0 != cudaSuccess) return e0;                                                                         \
        e0 = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, kern, p.sweep_warps * 32, smem);         \
        if (e0 != cudaSuccess) return e0;                                                                         \
    }
    BILUK_BS_DISPATCH(p.bs, OCC)
#undef OCC
    return cudaSuccess;
}

cudaError_t launch_spmv(const Op &o, const double *x, double *y, const int *skip, cudaStream_t s) {
    const int64_t ntiles = o.ntiles;
    if (ntiles == 0) return cudaSuccess;
    const int threads = 256;
    int64_t grid = (ntiles + (threads / 32) - 1) / (threads / 32);
    const int64_t cap = int64_t(o.num_sms) * 8;
    if (grid > cap) grid = cap;
    const TileMeta *meta = reinterpret_cast<const TileMeta *>(o.ws + o.off.meta);
    const unsigned char *rec = o.ws + o.off.rec;
#define SPMV_LAUNCH(BS) spmv_kernel<BS><<<unsigned(grid), threads, 0, s>>>(o.n, ntiles, meta, rec, x, y, skip);
    BILUK_BS_DISPATCH(o.bs, SPMV_LAUNCH)
#undef SPMV_LAUNCH
    return cudaGetLastError();
}

}  // namespace biluk
