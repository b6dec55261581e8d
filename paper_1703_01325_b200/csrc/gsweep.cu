// The grid sweep (engine 2): apply_preconditioner (trisolve.py:121-182)
//   L y = b,  z = D^-1 y,  U' x = z
// for ILU(0) of a 7-point block stencil on a natural-order nx x ny x nz grid
// (the headline configuration).  Layout and roles: biluk_internal.h (GSweep).
//
// One persistent cooperative launch, one CTA per (y, z) column part:
//   * 128 COMPUTE threads, thread t owns column t of its part.  Per level
//     (= record) a thread forms its row off the chain from its own previous
//     result (the x -/+ 1 neighbour) and the streamed blocks, then, after one
//     named barrier, adds the y and z neighbours' previous results (shared
//     memory, double-buffered) or, on a part face, the rows other parts
//     published (halo ring), and publishes: shared memory for its neighbours,
//     the natural-order y (L; read back by the U' sweep) or x (U'), and the
//     parity-tagged vector when a neighbouring part reads the row.
//   * one PRODUCER warp streams the part's records (one per level, L then U')
//     into a ring of fixed slots with cp.async.bulk on mbarriers.
//   * GS_HW HALO warps, warp w serving records w, w + GS_HW, ...: lane e
//     polls halo entry e (a row of a neighbouring part, one level back) until
//     its parity tag is current and stores it into the halo ring slot of the
//     record.  GS_HW records are polled concurrently, so the level rate is
//     not bounded by one L2 round trip per level.
// The inputs (b for L, y for U') of the row a thread handles GS_D records
// later are prefetched with cp.async into shared memory.
// Every CTA walks its levels in increasing order and every dependency lies
// one level back, so the CTA holding the lowest unfinished level is never
// blocked (no deadlock), exactly as in the partitioned sweep.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "biluk_internal.h"
#include "device_util.cuh"
#include "kernels.cuh"

namespace biluk {

using namespace dev;

namespace {

constexpr int GS_NC = 128;   // threads of a compute group = columns per part at most
constexpr int GS_G = 3;      // compute groups (round-robin over records)
constexpr int GS_HW = 3;     // halo warps
constexpr int GS_THREADS = GS_G * GS_NC + 32 + 32 * GS_HW;
constexpr int GS_D = 2;      // input prefetch depth (records of one group)
constexpr int GS_H = 16;     // halo ring slots (records)
constexpr int GS_K = 8;      // record ring slots at most
constexpr int GS_NE = 32;    // halo entries per part at most
constexpr int GS_PF = 3;     // records pulled into L2 ahead of their bulk copy

__device__ __forceinline__ void g_mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync_(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive_(int id, int threads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void g_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void g_cp_async_8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void g_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void g_cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void g_cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// bounded wait: false once the sweep is aborted or the wait timed out (which
// aborts it: sticky BILUK_ETIMEOUT)
__device__ __forceinline__ bool g_timed_out(uint64_t &t0, uint32_t &spins, const GSweepArgs &a) {
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
__device__ __forceinline__ bool g_wait(uint64_t *bar, uint32_t phase, int *abort_flag, const GSweepArgs &a) {
    uint64_t t0 = 0;
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, phase)) {
        if (*reinterpret_cast<volatile int *>(abort_flag)) return false;
        if (g_timed_out(t0, spins, a)) {
            *reinterpret_cast<volatile int *>(abort_flag) = 1;
            return false;
        }
    }
    return true;
}

}  // namespace

// ===========================================================================
// the sweep
// ===========================================================================
template <int BS>
__global__ void __launch_bounds__(GS_THREADS, 1) gsweep_kernel(const GSweepArgs a) {
    constexpr int BS2 = BS * BS;
    constexpr int TVS = tag_stride(BS);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full_bar[GS_K];    // record landed
    __shared__ __align__(8) uint64_t empty_bar[GS_K];   // record consumed (every compute thread)
    __shared__ __align__(8) uint64_t hfull[GS_H];       // halo values of a record stored (every lane of its halo warp)
    __shared__ __align__(8) uint64_t hempty[GS_H];      // halo slot consumed (every compute thread)
    __shared__ __align__(8) uint64_t ldone;             // every compute thread's y stores are done
    __shared__ int abort_flag;
    __shared__ int last_cta;
    if (a.skip_flag && ld_relaxed_s32(a.skip_flag) != 0) return;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const GPart pt = a.parts[blockIdx.x];
    const int nrec = pt.nl + pt.nu;
    const int K = a.kslots;
    const int64_t nx = a.nx, ny = a.ny, nz = a.nz;
    const int wy = pt.y1 - pt.y0, wz = pt.z1 - pt.z0;
    const int s0 = pt.y0 + pt.z0;                                    // first L level of the part
    const int u0 = int(ny - pt.y1) + int(nz - pt.z1);                // first U' level
    const uint32_t par = ld_relaxed_u32(&a.st->epoch) & 1u;
    // halo entries: L -- the y0-1 face (one per z), then the z0-1 face (one per y);
    // U' -- the y1 face, then the z1 face
    const int hzL = pt.y0 > 0 ? wz : 0, hzU = pt.y1 < ny ? wz : 0;
    const int neL = hzL + (pt.z0 > 0 ? wy : 0), neU = hzU + (pt.z1 < nz ? wy : 0);
    const int ne = neL > neU ? neL : neU;

    double *val = reinterpret_cast<double *>(smem);                  // [2][BS][GS_NC]
    double *inp = val + 2 * BS * GS_NC;                              // [GS_G][GS_D][BS][GS_NC]
    double *halo = inp + GS_G * GS_D * BS * GS_NC;                   // [GS_H][BS][GS_NE]
    unsigned char *ring = reinterpret_cast<unsigned char *>(halo + GS_H * BS * GS_NE);

    if (tid == 0) {
        for (int s = 0; s < GS_K; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, GS_NC);
        }
        for (int h = 0; h < GS_H; ++h) {
            mbar_init(hfull + h, 32);   // every lane of the serving halo warp
            mbar_init(hempty + h, GS_NC);
        }
        mbar_init(&ldone, GS_G * GS_NC);
        abort_flag = 0;
        fence_mbar_init();
    }
    for (int x = tid; x < 2 * BS * GS_NC; x += blockDim.x) val[x] = 0.0;
    __syncthreads();

    constexpr int GS_CW = GS_G * GS_NC / 32;   // compute warps; then the producer, then the halo warps
    if (warp == GS_CW) {
        // ======================= producer: the record stream =====================
        // lane l holds the descriptor of record base + l (a window of 32);
        // lane 0 issues the copies, pulling records GS_PF ahead into L2
        const uint64_t pol = policy_evict_first();
        const GRec *rec = a.recs + pt.rec0;
        long long w_off = 0;
        int w_bytes = 0;
        auto load_win = [&](int base) {
            const int j = base + lane;
            if (j < nrec) {
                const GRec ri = rec[j];
                w_off = ri.off;
                w_bytes = ri.bytes;
            }
        };
        load_win(0);
        if (lane < GS_PF && lane < nrec) g_prefetch_l2(a.stream + w_off, uint32_t(w_bytes));
        int issued = 0;
        for (; issued < nrec; ++issued) {
            if (issued > 0 && (issued & 31) == 0) load_win(issued);
            const int jl = issued & 31, pj = jl + GS_PF;
            const long long off = __shfl_sync(0xffffffffu, w_off, jl);
            const int bytes = __shfl_sync(0xffffffffu, w_bytes, jl);
            const long long poff = __shfl_sync(0xffffffffu, w_off, pj & 31);
            const int pbytes = __shfl_sync(0xffffffffu, w_bytes, pj & 31);
            const int slot = issued % K;
            int ok = 1;
            if (lane == 0 && issued >= K) ok = g_wait(empty_bar + slot, uint32_t(issued / K - 1) & 1u, &abort_flag, a);
            if (!__shfl_sync(0xffffffffu, ok, 0)) break;
            if (lane == 0) {
                mbar_expect_tx(full_bar + slot, uint32_t(bytes));
                bulk_g2s(ring + size_t(slot) * a.slot_bytes, a.stream + off, uint32_t(bytes), full_bar + slot, pol);
                if (a.trace) a.trace[size_t(pt.rec0 + issued) * 8 + 0] = globaltimer();
                if (pj < 32 && issued + GS_PF < nrec) g_prefetch_l2(a.stream + poff, uint32_t(pbytes));
            }
            __syncwarp();
        }
        // never leave the CTA with copies in flight into its shared memory
        if (lane == 0)
            for (int r = issued - K > 0 ? issued - K : 0; r < issued; ++r) mbar_wait(full_bar + r % K, uint32_t(r / K) & 1u);
    } else if (warp > GS_CW) {
        // ======================= halo warps =======================================
        const int hw = warp - GS_CW - 1;
        const bool has = lane < ne;
        for (int r = hw; r < nrec && ne > 0; r += GS_HW) {
            const int h = r % GS_H, k = r / GS_H;
            if (k > 0 && !g_wait(hempty + h, uint32_t(k - 1) & 1u, &abort_flag, a)) break;
            bool ok = true;
            if (has) {
                const bool up = r >= pt.nl;
                // the halo column of entry `lane` and its row one level back
                int64_t yh = -1, zh = -1;
                if (!up) {
                    if (lane < hzL) {
                        yh = pt.y0 - 1;
                        zh = pt.z0 + lane;
                    } else if (lane < neL) {
                        yh = pt.y0 + (lane - hzL);
                        zh = pt.z0 - 1;
                    }
                } else {
                    if (lane < hzU) {
                        yh = pt.y1;
                        zh = pt.z0 + lane;
                    } else if (lane < neU) {
                        yh = pt.y0 + (lane - hzU);
                        zh = pt.z1;
                    }
                }
                if (yh >= 0) {
                    int64_t x;
                    if (!up) {
                        x = int64_t(s0 + r - 1) - (yh + zh);
                    } else {
                        const int64_t u = int64_t(u0 + (r - pt.nl) - 1) - ((ny - 1 - yh) + (nz - 1 - zh));
                        x = nx - 1 - u;
                    }
                    if (x >= 0 && x < nx) {
                        const int64_t i = (zh * ny + yh) * nx + x;
                        const double *src = (up ? a.x_t : a.y_t) + size_t(i) * TVS;
                        double w[BS + 1];
                        ld_tagged<BS>(src, w);
                        uint64_t t0 = 0;
                        uint32_t spins = 0;
                        while (!row_ready<BS>(w, par)) {
                            if (*reinterpret_cast<volatile int *>(&abort_flag) || g_timed_out(t0, spins, a)) {
                                *reinterpret_cast<volatile int *>(&abort_flag) = 1;
                                ok = false;
                                break;
                            }
                            ld_tagged<BS>(src, w);
                        }
                        if (ok) {
                            double v[BS];
                            untag_row<BS>(w, v);
#pragma unroll
                            for (int c = 0; c < BS; ++c) halo[(h * BS + c) * GS_NE + lane] = v[c];
                        }
                    }
                }
            }
            // every lane releases its own stores (one arrival per lane)
            if (lane == 0 && a.trace) a.trace[size_t(pt.rec0 + r) * 8 + 6] = globaltimer();
            g_mbar_arrive(hfull + h);
            if (__any_sync(0xffffffffu, !ok)) break;
        }
    } else {
        // ======================= compute groups ====================================
        // group g takes records g, g + GS_G, ...; thread t of every group owns
        // column t.  Off the chain a group waits for its record, stages the
        // three neighbour blocks and the row's input term; on the chain -- a
        // named-barrier hand-over from the previous record's group -- it reads
        // the previous level's results (its own column: the x -/+ 1 neighbour;
        // the y and z neighbours or the halo), finishes the row, stores it for
        // the next level and hands over; the global stores follow off the chain.
        const int grp = warp / (GS_NC / 32), t = tid % GS_NC;
        const bool col = t < pt.ncols;
        int64_t y = 0, z = 0;
        if (col) {
            const int32_t yz = a.cols[size_t(blockIdx.x) * GS_NC + t];
            y = yz >> 16;
            z = yz & 0xffff;
        }
        const int d = int(y + z), du = int((ny - 1 - y) + (nz - 1 - z));
        // neighbour sources: >= 0 a column of this part, < -1 halo entry -(e + 2), -1 none
        auto find_col = [&](int64_t yy, int64_t zz) -> int {
            for (int q = 0; q < pt.ncols; ++q)
                if (a.cols[size_t(blockIdx.x) * GS_NC + q] == int32_t((yy << 16) | zz)) return q;
            return -1;
        };
        int nyL = -1, nzL = -1, nyU = -1, nzU = -1;
        if (col) {
            if (y > pt.y0) nyL = find_col(y - 1, z);
            else if (pt.y0 > 0) nyL = -(int(z - pt.z0) + 2);
            if (z > pt.z0) nzL = find_col(y, z - 1);
            else if (pt.z0 > 0) nzL = -(hzL + int(y - pt.y0) + 2);
            if (y < pt.y1 - 1) nyU = find_col(y + 1, z);
            else if (pt.y1 < ny) nyU = -(int(z - pt.z0) + 2);
            if (z < pt.z1 - 1) nzU = find_col(y, z + 1);
            else if (pt.z1 < nz) nzU = -(hzU + int(y - pt.y0) + 2);
        }
        const bool pubL = col && ((y == pt.y1 - 1 && pt.y1 < ny) || (z == pt.z1 - 1 && pt.z1 < nz));
        const bool pubU = col && ((y == pt.y0 && pt.y0 > 0) || (z == pt.z0 && pt.z0 > 0));
        // the row of this column at record r (-1: none)
        auto row_of = [&](int r) -> int64_t {
            if (!col) return -1;
            if (r < pt.nl) {
                const int64_t x = int64_t(s0 + r) - d;
                return (x >= 0 && x < nx) ? (z * ny + y) * nx + x : -1;
            }
            const int64_t u = int64_t(u0 + (r - pt.nl)) - du;
            return (u >= 0 && u < nx) ? (z * ny + y) * nx + (nx - 1 - u) : -1;
        };
        // input prefetch (this group's own record sequence, GS_D deep): b (L)
        // / y (U') of the row at record r into the group's slot
        double *ginp = inp + size_t(grp) * GS_D * BS * GS_NC;
        auto islot = [&](int r) { return ((r - grp) / GS_G) % GS_D; };
        auto prefetch = [&](int r) {
            const int64_t i = row_of(r);
            if (i >= 0) {
                const double *src = (r < pt.nl ? a.b : a.y) + size_t(i) * BS;
                double *dst = ginp + size_t(islot(r)) * BS * GS_NC + t;
#pragma unroll
                for (int c = 0; c < BS; ++c) g_cp_async_8(dst + c * GS_NC, src + c);
            }
            g_cp_commit();
        };
        // the first record of this group in [from, to), or to
        auto first_of = [&](int from) { return from + ((grp - from % GS_G) + GS_G) % GS_G; };
        for (int r = grp, j = 0; r < pt.nl && j < GS_D; r += GS_G, ++j) prefetch(r);
        const int uf = first_of(pt.nl);   // this group's first U' record
        // the U' inputs are the y rows every group stored in the L sweep: each
        // thread arrives on `ldone` after its last L stores (generic stores,
        // then fence.proxy.async for the copies), and a group waits on it
        // before its first U' input copies
        bool ldone_arrived = false;
        auto arrive_ldone = [&]() {
            __threadfence_block();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            g_mbar_arrive(&ldone);
            ldone_arrived = true;
        };
        if (grp >= pt.nl) arrive_ldone();   // a group without L records
        for (int r = grp; r < nrec; r += GS_G) {
            const bool up = r >= pt.nl;
            if (r == uf) {
                if (!g_wait(&ldone, 0u, &abort_flag, a)) *reinterpret_cast<volatile int *>(&abort_flag) = 1;
                for (int j = uf, m = 0; j < nrec && m < GS_D; j += GS_G, ++m) prefetch(j);
            }
            const int slot = r % K, h = r % GS_H;
            unsigned long long *tr = (a.trace && t == 0) ? a.trace + size_t(pt.rec0 + r) * 8 : nullptr;
            long long *dbg = (a.trace && t == 0 && pt.rec0 + r < 16384)
                                 ? reinterpret_cast<long long *>(a.trace) + size_t(a.nrec_total + pt.rec0 + r) * 8
                                 : nullptr;
            if (dbg) dbg[0] = clock64();
            bool ok = g_wait(full_bar + slot, uint32_t(r / K) & 1u, &abort_flag, a);
            if (dbg) dbg[1] = clock64();
            // inputs of record r: this group's later prefetches may stay in flight
            const int seg_end = up ? nrec : pt.nl;
            if (r + GS_G * (GS_D - 1) < seg_end) g_cp_wait<GS_D - 1>();
            else g_cp_wait_all();
            const unsigned char *rb = ring + size_t(slot) * a.slot_bytes;
            const int4 hdr = *reinterpret_cast<const int4 *>(rb);
            const double *vb = reinterpret_cast<const double *>(rb + 16);
            const int R = hdr.z;
            const int q = t - hdr.y;
            const bool act = ok && col && q >= 0 && q < hdr.x;
            double acc[BS];
            double b0[BS2], b1[BS2], b2[BS2];
            if (act) {
                const double *in = ginp + size_t(islot(r)) * BS * GS_NC + t;
                const double *bl = vb + (up ? BS2 * R : 0) + q;   // the three neighbour blocks
                if (up) {
#pragma unroll
                    for (int rr = 0; rr < BS; ++rr) {
                        double sacc = 0.0;
#pragma unroll
                        for (int c = 0; c < BS; ++c) sacc = fma(vb[size_t(c * BS + rr) * R + q], in[c * GS_NC], sacc);
                        acc[rr] = sacc;
                    }
                } else {
#pragma unroll
                    for (int rr = 0; rr < BS; ++rr) acc[rr] = in[rr * GS_NC];
                }
#pragma unroll
                for (int e = 0; e < BS2; ++e) {
                    b0[e] = bl[size_t(e) * R];
                    b1[e] = bl[size_t(BS2 + e) * R];
                    b2[e] = bl[size_t(2 * BS2 + e) * R];
                }
            }
            if (dbg) dbg[2] = clock64();
            if (ok && ne > 0) ok = g_wait(hfull + h, uint32_t(r / GS_H) & 1u, &abort_flag, a);
            if (!ok) *reinterpret_cast<volatile int *>(&abort_flag) = 1;
            if (dbg) dbg[3] = clock64();
            // ---- the chain: record r-1's group has stored the previous level
            if (r > 0) named_bar_sync_(1 + grp, 2 * GS_NC);
            if (dbg) dbg[4] = clock64();
            const bool aborted = *reinterpret_cast<volatile int *>(&abort_flag) != 0;
            if (!aborted && act) {
                const int n1 = up ? nyU : nyL, n2 = up ? nzU : nzL;
                const double *vp = val + size_t((r - 1) & 1) * BS * GS_NC;
                const double *hp = halo + size_t(h) * BS * GS_NE;
                double v0[BS], v1[BS], v2[BS];
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    v0[c] = vp[c * GS_NC + t];
                    v1[c] = n1 >= 0 ? vp[c * GS_NC + n1] : (n1 < -1 ? hp[c * GS_NE + (-n1 - 2)] : 0.0);
                    v2[c] = n2 >= 0 ? vp[c * GS_NC + n2] : (n2 < -1 ? hp[c * GS_NE + (-n2 - 2)] : 0.0);
                }
#pragma unroll
                for (int rr = 0; rr < BS; ++rr) {
                    double s0v = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
                    for (int c = 0; c < BS; ++c) {
                        s0v = fma(b0[c * BS + rr], v0[c], s0v);
                        s1 = fma(b1[c * BS + rr], v1[c], s1);
                        s2 = fma(b2[c * BS + rr], v2[c], s2);
                    }
                    acc[rr] -= (s0v + s1) + s2;
                }
                double *vn = val + size_t(r & 1) * BS * GS_NC + t;
#pragma unroll
                for (int c = 0; c < BS; ++c) vn[c * GS_NC] = acc[c];
            }
            // hand the level over (always, so no group waits forever on an abort)
            if (r + 1 < nrec) named_bar_arrive_(1 + (grp + 1) % GS_G, 2 * GS_NC);
            if (dbg) dbg[5] = clock64();
            if (aborted) {
                if (!ldone_arrived) arrive_ldone();
                break;
            }
            // ---- off the chain: global stores, releases, the next prefetch
            if (act) {
                const int64_t i = row_of(r);
                if (!up) {
#pragma unroll
                    for (int c = 0; c < BS; ++c) a.y[size_t(i) * BS + c] = acc[c];
                    if (pubL) st_tagged<BS>(a.y_t + size_t(i) * TVS, acc, par);
                } else {
                    if (a.out) {
#pragma unroll
                        for (int c = 0; c < BS; ++c) a.out[size_t(i) * BS + c] = acc[c];
                    }
                    if (pubU) st_tagged<BS>(a.x_t + size_t(i) * TVS, acc, par);
                }
            }
            g_mbar_arrive(empty_bar + slot);
            if (ne > 0) g_mbar_arrive(hempty + h);
            if (!up && r + GS_G >= pt.nl) arrive_ldone();   // this thread's last L record
            if (dbg) dbg[6] = clock64();
            const int nx_r = r + GS_G * GS_D;   // this group's record GS_D ahead, same sweep
            if (nx_r < (up ? nrec : pt.nl)) prefetch(nx_r);
            if (dbg) dbg[7] = clock64();
            if (tr) {   // (globaltimer reads cost hundreds of cycles: one per record, at its end)
                tr[5] = globaltimer();
                tr[7] = uint64_t(up ? 1 : 0) | (uint64_t(up ? u0 + r - pt.nl : s0 + r) << 10);
            }
        }
        g_cp_wait_all();
    }
    // the last CTA to finish advances the epoch (every CTA read it at entry)
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        last_cta = atomicAdd(&a.st->done_ctas, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last_cta && tid == 0) {
        __threadfence();
        a.st->done_ctas = 0;
        __threadfence();
        atomicAdd(&a.st->epoch, 1u);
    }
}

// ===========================================================================
// pack: the record stream from the factored values (L blocks verbatim, U' =
// D^-1 U after the split, D^-1); one CTA per record
// ===========================================================================
template <int BS>
__global__ void gpack_kernel(const GPart *__restrict__ parts, int P, const GRec *__restrict__ recs,
                             const int32_t *__restrict__ rec_lo, const int32_t *__restrict__ cols, int64_t nx,
                             int64_t ny, int64_t nz, const int32_t *__restrict__ p_rp, const int32_t *__restrict__ p_ci,
                             const double *__restrict__ pvals, const double *__restrict__ dinv,
                             unsigned char *__restrict__ stream) {
    constexpr int BS2 = BS * BS;
    __shared__ int64_t slot_of[3][GS_NC];
    __shared__ int64_t row_of[GS_NC];
    const int r = blockIdx.x;
    int c = 0;
    {
        int lo = 0, hi = P - 1;   // the part holding record r
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (parts[mid].rec0 <= r) lo = mid;
            else hi = mid - 1;
        }
        c = lo;
    }
    const GPart pt = parts[c];
    const int rl = r - pt.rec0;
    const bool up = rl >= pt.nl;
    const int level = up ? int(ny - pt.y1) + int(nz - pt.z1) + (rl - pt.nl) : pt.y0 + pt.z0 + rl;
    const GRec ri = recs[r];
    const int nr = ri.nrows, R = (nr + 1) & ~1, lo = rec_lo[r];
    const int64_t nxy = nx * ny;
    for (int q = threadIdx.x; q < R; q += blockDim.x) {
        int64_t i = -1;
        int64_t nb[3] = {-1, -1, -1};
        if (q < nr) {
            const int32_t yz = cols[size_t(c) * GS_NC + lo + q];
            const int64_t y = yz >> 16, z = yz & 0xffff;
            int64_t x;
            if (!up) {
                x = level - (y + z);
                i = (z * ny + y) * nx + x;
                if (x > 0) nb[0] = i - 1;
                if (y > 0) nb[1] = i - nx;
                if (z > 0) nb[2] = i - nxy;
            } else {
                x = nx - 1 - (level - ((ny - 1 - y) + (nz - 1 - z)));
                i = (z * ny + y) * nx + x;
                if (x < nx - 1) nb[0] = i + 1;
                if (y < ny - 1) nb[1] = i + nx;
                if (z < nz - 1) nb[2] = i + nxy;
            }
        }
        row_of[q] = i;
        for (int k = 0; k < 3; ++k) {
            int64_t sl = -1;
            if (nb[k] >= 0)
                for (int32_t e = p_rp[i]; e < p_rp[i + 1]; ++e)
                    if (p_ci[e] == nb[k]) sl = e;
            slot_of[k][q] = sl;
        }
    }
    __syncthreads();
    unsigned char *dst = stream + ri.off;
    if (threadIdx.x == 0) *reinterpret_cast<int4 *>(dst) = make_int4(nr, lo, R, 0);
    double *v = reinterpret_cast<double *>(dst + 16);
    if (up) {
        for (int e = threadIdx.x; e < BS2 * R; e += blockDim.x) {
            const int el = e / R, q = e - el * R;
            v[e] = row_of[q] >= 0 ? dinv[row_of[q] * BS2 + el] : 0.0;
        }
        v += BS2 * R;
    }
    for (int e = threadIdx.x; e < 3 * BS2 * R; e += blockDim.x) {
        const int k = e / (BS2 * R), rem = e - k * BS2 * R, el = rem / R, q = rem - el * R;
        const int64_t sl = slot_of[k][q];
        v[e] = sl >= 0 ? pvals[sl * BS2 + el] : 0.0;
    }
}

#define GS_BS_DISPATCH(bs, F)     \
    switch (bs) {                 \
        case 1: F(1); break;      \
        case 2: F(2); break;      \
        case 3: F(3); break;      \
        case 4: F(4); break;      \
        default: return cudaErrorInvalidValue; \
    }

size_t gsweep_smem_bytes(const Plan &p) {
    const GSweep &gs = p.gs;
    return size_t(2 + GS_G * GS_D) * p.bs * GS_NC * 8 + size_t(GS_H) * p.bs * GS_NE * 8 +
           size_t(gs.kslots) * gs.slot_bytes;
}

static cudaError_t gsweep_fn(const Plan &p, const void **fn) {
#define GS_FN(BS) *fn = reinterpret_cast<const void *>(gsweep_kernel<BS>);
    GS_BS_DISPATCH(p.bs, GS_FN)
#undef GS_FN
    return cudaSuccess;
}

cudaError_t launch_gsweep(const Plan &p, const GSweepArgs &a, cudaStream_t s) {
    const size_t smem = gsweep_smem_bytes(p);
    const void *fn = nullptr;
    cudaError_t e = gsweep_fn(p, &fn);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    void *args[] = {const_cast<GSweepArgs *>(&a)};
    e = cudaLaunchCooperativeKernel(fn, dim3(p.gs.P), dim3(GS_THREADS), args, smem, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t gsweep_occupancy(const Plan &p, int *blocks_per_sm) {
    const size_t smem = gsweep_smem_bytes(p);
    const void *fn = nullptr;
    cudaError_t e = gsweep_fn(p, &fn);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, GS_THREADS, smem);
}

cudaError_t launch_gpack(const Plan &p, cudaStream_t s) {
    const GSweep &gs = p.gs;
    const int nrec = int(gs.rec.size());
    if (nrec == 0) return cudaSuccess;
    const GPart *parts = reinterpret_cast<const GPart *>(p.ws + p.off.gs_part);
    const GRec *recs = reinterpret_cast<const GRec *>(p.ws + p.off.gs_rec);
    const int32_t *lo = reinterpret_cast<const int32_t *>(p.ws + p.off.gs_lo);
    const int32_t *cols = reinterpret_cast<const int32_t *>(p.ws + p.off.gs_cols);
    const int32_t *rp = reinterpret_cast<const int32_t *>(p.ws + p.off.p_rp);
    const int32_t *ci = reinterpret_cast<const int32_t *>(p.ws + p.off.p_ci);
    const double *pv = reinterpret_cast<const double *>(p.ws + p.off.pvals);
    const double *dv = reinterpret_cast<const double *>(p.ws + p.off.dinv);
    unsigned char *st = p.ws + p.off.gs_stream;
#define GPACK_LAUNCH(BS) \
    gpack_kernel<BS><<<nrec, 256, 0, s>>>(parts, gs.P, recs, lo, cols, gs.nx, gs.ny, gs.nz, rp, ci, pv, dv, st);
    GS_BS_DISPATCH(p.bs, GPACK_LAUNCH)
#undef GPACK_LAUNCH
    return cudaGetLastError();
}

// ===========================================================================
// host planner
// ===========================================================================
int plan_gsweep(Plan &p, int num_sms, size_t smem_per_block) {
    GSweep &gs = p.gs;
    gs = GSweep{};
    const int bs = p.bs, bs2 = bs * bs;
    if (p.k != 0 || bs < 1 || bs > 4) return BILUK_EUNSUPPORTED;
    int64_t g[3] = {0, 0, 0};
    if (!detect_grid(p, g)) return BILUK_EUNSUPPORTED;
    const int64_t nx = g[0], ny = g[1], nz = g[2], nxy = nx * ny;
    if (ny > 32767 || nz > 32767 || nx > (int64_t(1) << 30)) return BILUK_EUNSUPPORTED;
    // the pattern of every row must lie in the 7-point stencil
    for (int64_t i = 0; i < p.n; ++i) {
        const int64_t x = i % nx, y = (i / nx) % ny, z = i / nxy;
        for (int32_t t = p.p_rp[i]; t < p.p_rp[i + 1]; ++t) {
            const int64_t dlt = int64_t(p.p_ci[t]) - i;
            const bool ok = dlt == 0 || (dlt == -1 && x > 0) || (dlt == 1 && x < nx - 1) || (dlt == -nx && y > 0) ||
                            (dlt == nx && y < ny - 1) || (dlt == -nxy && z > 0) || (dlt == nxy && z < nz - 1);
            if (!ok) return BILUK_EUNSUPPORTED;
        }
    }
    Partition part;
    partition_grid_columns(p, num_sms, g, part);
    const int py = part.split[0], pz = part.split[1], P = py * pz;
    gs.P = P;
    gs.py = py;
    gs.pz = pz;
    gs.nx = nx;
    gs.ny = ny;
    gs.nz = nz;
    gs.part.resize(P);
    gs.cols.assign(size_t(P) * GS_NC, 0);
    int64_t off = 0;
    int64_t max_bytes = 0;
    for (int cz = 0; cz < pz; ++cz)
        for (int cy = 0; cy < py; ++cy) {
            const int c = cz * py + cy;
            GPart &pp = gs.part[c];
            // column j belongs to part floor(j * p / n): part a starts at ceil(a * n / p)
            pp.y0 = int32_t((int64_t(cy) * ny + py - 1) / py);
            pp.y1 = int32_t((int64_t(cy + 1) * ny + py - 1) / py);
            pp.z0 = int32_t((int64_t(cz) * nz + pz - 1) / pz);
            pp.z1 = int32_t((int64_t(cz + 1) * nz + pz - 1) / pz);
            const int wy = pp.y1 - pp.y0, wz = pp.z1 - pp.z0;
            if (wy < 1 || wz < 1 || wy * wz > GS_NC) return BILUK_EUNSUPPORTED;
            const int ne = std::max((pp.y0 > 0 ? wz : 0) + (pp.z0 > 0 ? wy : 0),
                                    (pp.y1 < ny ? wz : 0) + (pp.z1 < nz ? wy : 0));
            if (ne > GS_NE) return BILUK_EUNSUPPORTED;
            gs.ne = std::max(gs.ne, ne);
            std::vector<std::pair<int, int>> cl;   // (y, z) by (y + z, y)
            for (int y = pp.y0; y < pp.y1; ++y)
                for (int z = pp.z0; z < pp.z1; ++z) cl.emplace_back(y, z);
            std::sort(cl.begin(), cl.end(), [](const std::pair<int, int> &u, const std::pair<int, int> &v) {
                return u.first + u.second != v.first + v.second ? u.first + u.second < v.first + v.second
                                                                 : u.first < v.first;
            });
            pp.ncols = int32_t(cl.size());
            std::vector<int> dcol(cl.size());
            for (size_t q = 0; q < cl.size(); ++q) {
                gs.cols[size_t(c) * GS_NC + q] = (cl[q].first << 16) | cl[q].second;
                dcol[q] = cl[q].first + cl[q].second;
            }
            auto count_below = [&](int64_t dd) {   // columns with d < dd
                return int(std::lower_bound(dcol.begin(), dcol.end(), dd) - dcol.begin());
            };
            pp.rec0 = int32_t(gs.rec.size());
            pp.nl = (wy - 1) + (wz - 1) + int32_t(nx);
            pp.nu = pp.nl;
            for (int j = 0; j < pp.nl + pp.nu; ++j) {
                int lo, hi;
                const bool up = j >= pp.nl;
                if (!up) {
                    const int64_t s = pp.y0 + pp.z0 + j;   // active: d in [s - nx + 1, s]
                    lo = count_below(s - nx + 1);
                    hi = count_below(s + 1);
                } else {
                    const int64_t sg = (ny - pp.y1) + (nz - pp.z1) + (j - pp.nl);
                    const int64_t dlo = (ny + nz - 2) - sg;   // active: d in [dlo, dlo + nx - 1]
                    lo = count_below(dlo);
                    hi = count_below(dlo + nx);
                }
                const int nr = hi - lo, R = (nr + 1) & ~1;
                GRec ri{};
                ri.off = off;
                ri.nrows = nr;
                ri.bytes = int32_t(16 + int64_t(up ? 4 : 3) * bs2 * R * 8);
                ri.bytes = (ri.bytes + 15) & ~15;
                off += (ri.bytes + 127) & ~127;
                max_bytes = std::max<int64_t>(max_bytes, ri.bytes);
                gs.rec.push_back(ri);
                gs.rec_lo.push_back(lo);
            }
        }
    gs.stream_bytes = off;
    gs.slot_bytes = int32_t((max_bytes + 127) & ~int64_t(127));
    const int64_t fixed = int64_t(2 + GS_G * GS_D) * bs * GS_NC * 8 + int64_t(GS_H) * bs * GS_NE * 8;
    const int64_t budget = int64_t(smem_per_block) - 2048 - fixed;
    gs.kslots = int32_t(std::min<int64_t>(GS_K, budget / gs.slot_bytes));
    if (gs.kslots < 2) return BILUK_EUNSUPPORTED;
    return BILUK_OK;
}

}  // namespace biluk
