// The apply engine: a persistent, partitioned, sync-free sweep for
//   L y = b,  z = D^-1 y,  U' x = z      (apply_preconditioner, trisolve.py:121-182)
// and the device pack of its records from the factors.
//
// One CTA per part (grid columns for ILU(0), contiguous row ranges with fill;
// psweep_plan.cpp), all CTAs co-resident (cooperative launch).  A part's rows
// are cut into RECORDS (<= 128 rows of one level, L records then U' records).
// Inside a CTA:
//   * G COMPUTE GROUPS of 128 threads (G = 3 for ILU(0), 2 with fill) take
//     records round-robin, one thread per block row:
//       L :  y_i = b_i - sum_j L_ij y_j
//       U':  x_i = D_i^-1 y_i - sum_j U'_ij x_j
//     Off the chain, a group stages its next record (indices, b or D^-1 y,
//     the shared addresses of every dependency) and fetches the record's
//     dependencies held by other parts from the parity-tagged global vector
//     (tag-polled; the first load overlaps the staging).  On the chain -- a
//     named-barrier hand-over from the previous record's group -- it loads
//     the dependencies from shared memory (the part's vector ring or the
//     fetched values), forms the products and publishes the row to the ring,
//     to the tagged global vector (other parts poll it) and to y_u (L, the
//     U' input) or the caller's x (U').
//   * NP PRODUCER warps (record r served by producer r % NP, each in its
//     share of the data ring) stream records and their rows' inputs (b_perm /
//     y_u, position ordered) into shared memory with cp.async.bulk on
//     mbarriers, pulling records ahead into L2 with cp.async.bulk.prefetch.L2.
// Published rows go to the part's vector ring, to the parity-tagged global
// vector (only rows some record fetches: iarr bit 31) as exact tagged rows
// (tag_row), and to y_u (L) / the caller's x (U').
// Every CTA walks its rows in global level order, L then U', and every
// dependency has a lower level, so the CTA holding the lowest unfinished row
// is never blocked -- for any row-to-part assignment (no deadlock).
#include <cstdint>

#include "biluk_internal.h"
#include "device_util.cuh"
#include "kernels.cuh"

namespace biluk {

using namespace dev;

namespace {

constexpr int PS_NG = 128;            // threads per compute group (= rows per record)
// compute groups (round-robin over records) are a template parameter G: 2 or 3
// producer warps (record r served by producer r % NP) are a template
// parameter NP: 2, or 1 for ILU(2)+ where the freed registers stage blocks
constexpr int PS_PF = 2;              // records pulled into L2 ahead of their bulk copy (2 measured best of 0-32)
constexpr uint32_t PS_PUB = 0x80000000u;   // iarr bit: publish the row to the tagged vector

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int threads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// circular allocation of `sz` bytes in a ring of `cap` bytes whose oldest
// live allocation starts at `tail` (`live` allocations outstanding, the next
// free byte is `head`); returns the offset or -1
__device__ __forceinline__ int64_t ring_alloc(uint32_t &head, uint32_t tail, int live, uint32_t sz, uint32_t cap) {
    if (live == 0) {
        head = sz;
        return 0;
    }
    if (head > tail) {
        if (head + sz <= cap) {
            const uint32_t at = head;
            head += sz;
            return at;
        }
        if (sz <= tail) {
            head = sz;
            return 0;
        }
        return -1;
    }
    if (head < tail && head + sz <= tail) {
        const uint32_t at = head;
        head += sz;
        return at;
    }
    return -1;
}

// a tagged row of 4 words as one 256-bit load (others as ld_tagged)
template <int BS>
__device__ __forceinline__ void ld_tagged_wide(const double *p, double (&w)[BS + 1]) {
    if constexpr (BS + 1 == 4) {
        ld_relaxed_v4(p, w[0], w[1], w[2], w[3]);
    } else {
        ld_tagged<BS>(p, w);
    }
}
__device__ __forceinline__ bool ps_timed_out(uint64_t &t0, uint32_t &spins, const PSweepArgs &a) {
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

}  // namespace

__device__ __forceinline__ void cp_async_16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// non-blocking probe of an mbarrier phase (try_wait may suspend the thread)
__device__ __forceinline__ bool mbar_test_wait(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

// wait for an mbarrier phase; false if the sweep was aborted meanwhile or the
// wait exceeded the timeout (which then aborts the sweep: sticky status)
__device__ __forceinline__ bool mbar_wait_or_abort(uint64_t *bar, uint32_t phase, int *abort_flag, const PSweepArgs &a) {
    uint64_t t0 = 0;
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, phase)) {
        if (*reinterpret_cast<volatile int *>(abort_flag)) return false;
        if (ps_timed_out(t0, spins, a)) {
            *reinterpret_cast<volatile int *>(abort_flag) = 1;
            return false;
        }
    }
    return true;
}

template <int BS, int G, int NP>
__global__ void __launch_bounds__(G * PS_NG + 32 * NP, 1) psweep_kernel(const PSweepArgs a) {
    constexpr int PS_NW = G * PS_NG / 32;   // compute warps; then the two producers
    constexpr int BS2 = BS * BS;
    constexpr int VS = ps_vec_stride(BS);   // component planes of the vector ring
    constexpr int TVS = tag_stride(BS);     // tagged rows of y_t / x_t
    constexpr int K = PS_KSLOTS;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full_bar[K];    // record bytes + inputs landed (two bulk copies)
    __shared__ __align__(8) uint64_t empty_bar[K];   // record consumed (every thread of a compute group)
    __shared__ uint32_t slot_off[K];
    __shared__ __align__(8) uint64_t ldone_bar;      // every compute thread is past its last L record
    __shared__ int abort_flag;   // a wait timed out somewhere (the device status is sticky)
    __shared__ int last_cta;
    if (a.skip_flag && ld_relaxed_s32(a.skip_flag) != 0) return;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double *vring = reinterpret_cast<double *>(smem);
    unsigned char *dring = smem + align128(int64_t(a.ring_mask + 2) * VS * 8);   // the records start 128-aligned
    const int r0 = a.part_rec[blockIdx.x], nrec = a.part_rec[blockIdx.x + 1] - r0;
    const int nlrec = a.part_rec[gridDim.x + 1 + blockIdx.x];   // L records come first
    const uint32_t par = ld_relaxed_u32(&a.st->epoch) & 1u;

    if (tid == 0) {
        for (int s = 0; s < K; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, PS_NG);
        }
        mbar_init(&ldone_bar, G * PS_NG);
        abort_flag = 0;
        fence_mbar_init();
    }
    // vector ring, component-major: component c of slot k at vring[c * RS + k]; slot ring_mask+1 is zero
    const int RS = a.ring_mask + 2;
    for (int x = tid; x < VS; x += blockDim.x) vring[size_t(x) * RS + a.ring_mask + 1] = 0.0;
    __syncthreads();

    if (warp >= PS_NW && warp < PS_NW + NP) {
        // ============ producers: records into the data ring ==================
        // producer pp serves records pp, pp+NP, ... in its own share of the
        // ring.  Per record two bulk copies on one mbarrier: the record's bytes
        // and its rows' inputs (positions pos0 .. pos0+nr of b_perm for L, of
        // y_u for U' -- the latter only once this part's L sweep is complete).
        // Space is recycled in record order (empty barriers); records are
        // pulled into L2 ahead so the copies are short.
        const int pp = warp - PS_NW;
        const int nk = (nrec - pp + NP - 1) / NP;   // records of this producer: pp + NP k
        const uint32_t half = (a.data_bytes / NP) & ~15u;
        unsigned char *ring = dring + pp * half;
        const uint64_t pol = policy_evict_first();
        uint32_t dhead = 0;
        int oldest = 0;   // (own sequence) first record not yet known consumed
        int issued = 0;
        bool up_ready = false;
        // record descriptors in registers, two windows of 32 (lane l: own record base + l)
        uint64_t cur_off = 0, nxt_off = 0;
        uint32_t cur_bytes = 0, cur_foot = 0, cur_pm = 0, nxt_bytes = 0, nxt_foot = 0, nxt_pm = 0;
        uint32_t cur_nr = 0, nxt_nr = 0;
        auto fetch = [&](int k, uint64_t &off, uint32_t &bytes, uint32_t &foot, uint32_t &pos0u, uint32_t &nr) {
            const PRecInfo &ri = a.rec[r0 + pp + NP * k];
            off = ri.off;
            bytes = ri.bytes;
            foot = ri.foot;
            pos0u = uint32_t(ri.pos0) | (uint32_t(ri.level & 1) << 31);
            nr = uint32_t(ri.nrows);
        };
        auto wait_rec = [&](int rr) -> bool {   // own record rr consumed
            return mbar_wait_or_abort(empty_bar + rr % K, uint32_t(rr / K) & 1u, &abort_flag, a);
        };
        if (lane < nk) fetch(lane, cur_off, cur_bytes, cur_foot, cur_pm, cur_nr);
        if (32 + lane < nk) fetch(32 + lane, nxt_off, nxt_bytes, nxt_foot, nxt_pm, nxt_nr);
        constexpr int PFO = PS_PF / NP > 0 ? PS_PF / NP : 1;   // own records prefetched ahead
        for (int j = lane; j < PFO && j < nk; j += 32) bulk_prefetch_l2(a.recs + cur_off, cur_bytes);
        for (; issued < nk; ++issued) {
            if (issued > 0 && (issued & 31) == 0) {   // slide the window by 32 records
                cur_off = nxt_off;
                cur_bytes = nxt_bytes;
                cur_foot = nxt_foot;
                cur_pm = nxt_pm;
                cur_nr = nxt_nr;
                const int j = issued + 32 + lane;
                if (j < nk) fetch(j, nxt_off, nxt_bytes, nxt_foot, nxt_pm, nxt_nr);
            }
            const int jl = issued & 31;
            const uint64_t off = __shfl_sync(0xffffffffu, cur_off, jl);
            const uint32_t bytes = __shfl_sync(0xffffffffu, cur_bytes, jl);
            const uint32_t foot = __shfl_sync(0xffffffffu, cur_foot, jl);
            const uint32_t pm = __shfl_sync(0xffffffffu, cur_pm, jl);
            const uint32_t nr = __shfl_sync(0xffffffffu, cur_nr, jl);
            const bool up = pm >> 31;
            const uint32_t pos0 = pm & 0x7fffffffu;
            const int rr = pp + NP * issued;   // record index
            bool ok = true;
            if (up && !up_ready) {
                // y_u is written by this part's L sweep (generic proxy): every
                // compute thread issues fence.proxy.async after its last L
                // record and then arrives on ldone_bar, so this wait orders
                // every y_u store before the U' input bulk copies
                ok = mbar_wait_or_abort(&ldone_bar, 0u, &abort_flag, a);
                up_ready = true;
            }
            // wait for a free ring slot and room for the footprint in this half
            int64_t at = -1;
            while (ok) {
                if (issued - oldest >= K / NP) {
                    ok = wait_rec(pp + NP * oldest);
                    ++oldest;
                    continue;
                }
                const int live = issued - oldest;
                at = ring_alloc(dhead, live ? slot_off[(pp + NP * oldest) % K] - pp * half : 0, live, foot, half);
                if (at >= 0) break;
                ok = wait_rec(pp + NP * oldest);
                ++oldest;
            }
            if (!ok) break;
            const int si = rr % K;
            // pull a record ahead into L2 (no shared memory)
            const int pf = issued + PFO;
            const int pj = pf - (issued & ~31);   // index into the two windows
            const uint64_t pf_off = __shfl_sync(0xffffffffu, pj < 32 ? cur_off : nxt_off, pj & 31);
            const uint32_t pf_bytes = __shfl_sync(0xffffffffu, pj < 32 ? cur_bytes : nxt_bytes, pj & 31);
            // packed input rows: the copy starts at the 16-byte boundary at or
            // below the first row (head = 0 or 8 bytes) and ends on one
            const uint64_t in_src = uint64_t(pos0) * (BS * 8);
            const uint32_t head = uint32_t(in_src & 15u);
            const uint32_t in_bytes = (head + nr * uint32_t(BS * 8) + 15u) & ~15u;
            if (lane == 0) {
                slot_off[si] = uint32_t(at) + pp * half;
                mbar_expect_tx(full_bar + si, bytes + in_bytes);
                bulk_g2s(ring + at, a.recs + off, bytes, full_bar + si, pol);
                bulk_g2s(ring + at + bytes,
                         reinterpret_cast<const unsigned char *>(up ? a.y_u : a.b_perm) + (in_src - head), in_bytes,
                         full_bar + si, pol);
                if (pf < nk && pj < 64) bulk_prefetch_l2(a.recs + pf_off, pf_bytes);
                if (a.trace) a.trace[size_t(r0 + rr) * 8 + 0] = globaltimer();
            }
            __syncwarp();
        }
        // never leave the CTA with copies in flight into its shared memory
        for (int g = oldest; g < issued; ++g) mbar_wait(full_bar + (pp + NP * g) % K, uint32_t((pp + NP * g) / K) & 1u);
    } else {
        // ========================= compute warps ==============================
        // two groups of PS_NG threads take alternate records (ping-pong).  A
        // group prepares its next record while the other group computes:
        // header, the row's accumulator init (b, or D^-1 y), its first SR
        // blocks and the shared-memory addresses of their dependencies.  The
        // hand-over is a named-barrier arrive/sync, so the level chain only
        // carries [dependency loads -> products -> publish].
        constexpr int SR = BS <= 2 ? 6 : (BS <= 3 ? 3 : (BS <= 4 ? 2 : 1));
        const int grp = warp / (PS_NG / 32), gt = tid % PS_NG;
        // dependency addresses are byte offsets into the dynamic shared memory;
        // plain C++ accesses let the compiler overlap the loads (they stay
        // ordered against the barriers, which clobber memory)
        const uint32_t vring_s = 0;   // the vector ring starts the dynamic shared memory
        auto lds = [&](uint32_t off) -> double { return *reinterpret_cast<const double *>(smem + off); };
        auto sts = [&](uint32_t off, double v) { *reinterpret_cast<double *>(smem + off) = v; };
        bool ldone = false;   // arrived on ldone_bar (once per thread, before its first U' record)
        auto arrive_ldone = [&]() {
            fence_proxy_async_global();   // this thread's y_u stores, before the U' input bulk copies
            mbar_arrive(&ldone_bar);
            ldone = true;
        };
        for (int i = grp; i < nrec; i += G) {
            const int s = i % K;
            const uint32_t ph = uint32_t(i / K) & 1u;
            if (!ldone && i >= nlrec) arrive_ldone();
            if (!mbar_wait_or_abort(full_bar + s, ph, &abort_flag, a)) {
                // aborted: still pass the hand-over on, so no group waits forever
                if (i > 0) named_bar_sync(1 + grp, 2 * PS_NG);
                if (i + 1 < nrec) named_bar_arrive(1 + (grp + 1) % G, 2 * PS_NG);
                break;
            }
            // clock64 stamps of the stages for the first 16384 records (trace debug rows)
            unsigned long long *dbg =
                (a.trace && gt == 0 && r0 + i < 16384) ? a.trace + size_t(a.nrec_total + r0 + i) * 8 : nullptr;
            if (dbg) dbg[0] = clock64();
            if (a.trace && gt == 0) a.trace[size_t(r0 + i) * 8 + 1] = globaltimer();
            const unsigned char *rec = dring + slot_off[s];
            const PRecHdr h = *reinterpret_cast<const PRecHdr *>(rec);
            const int nr = h.nrows, S = h.S, ng = h.nglob;
            const bool up = h.flags & 1;
            const bool live = gt < nr;
            const int32_t *iarr = reinterpret_cast<const int32_t *>(rec + sizeof(PRecHdr));
            const int16_t *desc = reinterpret_cast<const int16_t *>(iarr + nr);   // two entries per word
            // block values as 32-bit shared byte offsets: element k of row q of
            // the record's blocks at vb_s + (k * nr + q) * 8 (k = slot * BS2 + e;
            // a U' record's D^-1 blocks precede them)
            const uint32_t vstr = uint32_t(nr) * 8u;
            const uint32_t vb_s = uint32_t(rec + h.vals_off - smem) + (up ? uint32_t(BS2) * vstr : 0u);
            const uint32_t vals_s = vb_s + uint32_t(gt) * 8u;
            const double *inp0 = reinterpret_cast<const double *>(rec + h.in_off + ((uint32_t(h.pos0) * (BS * 8)) & 15u));
            const uint32_t dep_s = uint32_t(rec + h.in_off - smem) + uint32_t(ps_in_bytes(BS, nr));
            // dependencies outside the ring: thread e fetches entry e (tag-polled);
            // the first load is issued here so its round trip overlaps the prep
            const int32_t *gpos = iarr + nr + (S * nr + 1) / 2;
            const double *gvec = up ? a.x_t : a.y_t;
            const bool dneed = gt < ng;
            double dval[BS + 1];
            if (dneed) ld_tagged_wide<BS>(gvec + size_t(gpos[gt]) * TVS, dval);
            // accumulator init of row q: b (L) or D^-1 y (U'), both off the chain
            auto init_acc = [&](int q, double (&acc)[BS]) {
                const double *inp = inp0 + size_t(q) * BS;
                if (up) {
                    const uint32_t dv_s = vb_s - uint32_t(BS2) * vstr + uint32_t(q) * 8u;
#pragma unroll
                    for (int r = 0; r < BS; ++r) {
                        double z = lds(dv_s + uint32_t(r) * vstr) * inp[0];
#pragma unroll
                        for (int c = 1; c < BS; ++c) z = fma(lds(dv_s + uint32_t(c * BS + r) * vstr), inp[c], z);
                        acc[r] = z;
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < BS; ++r) acc[r] = inp[r];
                }
            };
            // slots [from, S) of row q straight from shared memory, 4 at a time
            auto smem_slots = [&](int q, int from, double (&acc)[BS]) {
                for (int sl0 = from; sl0 < S; sl0 += 4) {
                    uint32_t ad[4], st[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int32_t dd = sl0 + u < S ? desc[(sl0 + u) * nr + q] : a.ring_mask + 1;
                        ad[u] = dd >= 0 ? vring_s + uint32_t(dd) * 8u : dep_s + uint32_t(-dd - 1) * 8u;
                        st[u] = dd >= 0 ? uint32_t(RS) * 8u : uint32_t(ng) * 8u;
                    }
                    double xv[4][BS];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int c = 0; c < BS; ++c) xv[u][c] = lds(ad[u] + uint32_t(c) * st[u]);
                    double p2[4][BS];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t vv_s = vb_s + uint32_t(q) * 8u + uint32_t((sl0 + u) * BS2) * vstr;
                        const bool on = sl0 + u < S;
#pragma unroll
                        for (int r = 0; r < BS; ++r) p2[u][r] = on ? lds(vv_s + uint32_t(r) * vstr) * xv[u][0] : 0.0;
#pragma unroll
                        for (int c = 1; c < BS; ++c)
#pragma unroll
                            for (int r = 0; r < BS; ++r)
                                if (on) p2[u][r] = fma(lds(vv_s + uint32_t(c * BS + r) * vstr), xv[u][c], p2[u][r]);
                    }
#pragma unroll
                    for (int r = 0; r < BS; ++r) acc[r] -= (p2[0][r] + p2[1][r]) + (p2[2][r] + p2[3][r]);
                }
            };
            // publish row q: the ring (this part's next levels), the tagged
            // global vector (other parts) and y_u (L) / the caller's x (U')
            auto publish = [&](int q, uint32_t iv, const double (&acc)[BS]) {
                const uint32_t rs = vring_s + uint32_t((h.seq0 + q) & a.ring_mask) * 8u;
#pragma unroll
                for (int r = 0; r < BS; ++r) sts(rs + uint32_t(r) * uint32_t(RS) * 8u, acc[r]);
                if (iv & PS_PUB) st_tagged<BS>((up ? a.x_t : a.y_t) + size_t(h.pos0 + q) * TVS, acc, par);
                const uint32_t idx = iv & ~PS_PUB;
                if (up) {
                    if (a.out) {
#pragma unroll
                        for (int r = 0; r < BS; ++r) a.out[size_t(idx) * BS + r] = acc[r];
                    }
                } else {
                    double *yu = a.y_u + size_t(idx) * BS;
#pragma unroll
                    for (int r = 0; r < BS; ++r) yu[r] = acc[r];
                }
            };
            double acc[BS];
            // staged slots: all SR with two groups or one producer; with three
            // groups and two producers (128 registers) one slot for b <= 4 and
            // the other blocks are read at the products
            constexpr int SV = (G == 2 || NP == 1) ? SR : (BS <= 4 ? 1 : 0);
            double v[SV > 0 ? SV : 1][BS2] = {};
            // element e of slot u's block of this thread's row (registers, or shared memory)
            auto vblk = [&](int u, int e) -> double {
                return u < SV ? v[u][e] : (u < S ? lds(vals_s + uint32_t(u * BS2 + e) * vstr) : 0.0);
            };
            uint32_t xa[SR];   // shared address of component 0 of each staged dependency
            uint32_t xs[SR];   // its component stride in bytes
            uint32_t idx = 0;   // iarr entry: L: the row's U' position; U': its natural row (| PS_PUB)
            // rows longer than the staged slots in a record of few rows: TPR
            // threads per row share its slots (strided) and sum by shuffles,
            // so the idle threads of a short record shorten the chain
            const int tpr = S > SR ? (nr <= 16 ? 8 : nr <= 32 ? 4 : nr <= 64 ? 2 : 1) : 1;
            const int tq = gt / tpr, tj = gt & (tpr - 1);   // split: row and slot lane
            const bool tlive = tq < nr;
            if (tpr > 1) {
#pragma unroll
                for (int r = 0; r < BS; ++r) acc[r] = 0.0;
                if (tlive && tj == 0) {
                    idx = uint32_t(iarr[tq]);
                    init_acc(tq, acc);
                }
            } else if (live) {
                idx = uint32_t(iarr[gt]);
                init_acc(gt, acc);
#pragma unroll
                for (int u = 0; u < SR; ++u) {
                    const int32_t d = u < S ? desc[u * nr + gt] : a.ring_mask + 1;
                    xa[u] = d >= 0 ? vring_s + uint32_t(d) * 8u : dep_s + uint32_t(-d - 1) * 8u;
                    xs[u] = d >= 0 ? uint32_t(RS) * 8u : uint32_t(ng) * 8u;
#pragma unroll
                    for (int e = 0; e < BS2; ++e)
                        if (u < SV) v[u][e] = u < S ? lds(vals_s + uint32_t(u * BS2 + e) * vstr) : 0.0;
                }
            }
            if (dbg) dbg[1] = clock64();
            if (a.trace && gt == 0) a.trace[size_t(r0 + i) * 8 + 2] = globaltimer();
            {
                auto fetch_dep = [&](int e, double (&dv)[BS + 1], bool loaded) {
                    const double *src = gvec + size_t(gpos[e]) * TVS;
                    if (!loaded) ld_tagged_wide<BS>(src, dv);
                    uint64_t t0 = 0;
                    uint32_t spins = 0;
                    while (!row_ready<BS>(dv, par)) {
                        if (ps_timed_out(t0, spins, a)) {
                            *reinterpret_cast<volatile int *>(&abort_flag) = 1;
                            break;
                        }
                        ld_tagged_wide<BS>(src, dv);
                    }
                    double v[BS];
                    untag_row<BS>(dv, v);
#pragma unroll
                    for (int q = 0; q < BS; ++q) sts(dep_s + uint32_t(q * ng + e) * 8u, v[q]);
                };
                if (dneed) fetch_dep(gt, dval, true);
                for (int e = gt + PS_NG; e < ng; e += PS_NG) {
                    double dv2[BS + 1];
                    fetch_dep(e, dv2, false);
                }
                if (a.trace && gt == 0) a.trace[size_t(r0 + i) * 8 + 3] = globaltimer();
                if (i == 0) named_bar_sync(1 + G + grp, PS_NG);   // the fetched values, to the whole group
            }
            if (a.trace && gt == 0) a.trace[size_t(r0 + i) * 8 + 4] = globaltimer();
            if (dbg) dbg[2] = clock64();
            // the other group has published record i-1
            if (i > 0) named_bar_sync(1 + grp, 2 * PS_NG);   // arrive of record i-1's group
            if (dbg) dbg[3] = clock64();
            if (*reinterpret_cast<volatile int *>(&abort_flag)) {
                if (i + 1 < nrec) named_bar_arrive(1 + (grp + 1) % G, 2 * PS_NG);   // pass it on
                break;
            }
            if (tpr > 1) {
                if (tlive) {
                    for (int u = tj; u < S; u += tpr) {
                        const int32_t d = desc[u * nr + tq];
                        const uint32_t ad = d >= 0 ? vring_s + uint32_t(d) * 8u : dep_s + uint32_t(-d - 1) * 8u;
                        const uint32_t st = d >= 0 ? uint32_t(RS) * 8u : uint32_t(ng) * 8u;
                        double x[BS];
#pragma unroll
                        for (int c = 0; c < BS; ++c) x[c] = lds(ad + uint32_t(c) * st);
                        const uint32_t vv_s = vb_s + uint32_t(tq) * 8u + uint32_t(u * BS2) * vstr;
                        double pu[BS];
#pragma unroll
                        for (int r = 0; r < BS; ++r) pu[r] = lds(vv_s + uint32_t(r) * vstr) * x[0];
#pragma unroll
                        for (int c = 1; c < BS; ++c)
#pragma unroll
                            for (int r = 0; r < BS; ++r) pu[r] = fma(lds(vv_s + uint32_t(c * BS + r) * vstr), x[c], pu[r]);
#pragma unroll
                        for (int r = 0; r < BS; ++r) acc[r] -= pu[r];
                    }
                }
                for (int o = tpr >> 1; o > 0; o >>= 1)
#pragma unroll
                    for (int r = 0; r < BS; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
                if (dbg) dbg[4] = clock64();
                if (tlive && tj == 0) publish(tq, idx, acc);
                if (dbg) dbg[5] = clock64();
            } else if (live) {
                // register-staged slots: every dependency load first, then the
                // products, summed as a tree and subtracted once
                double x[SR][BS];
#pragma unroll
                for (int u = 0; u < SR; ++u)
#pragma unroll
                    for (int c = 0; c < BS; ++c) x[u][c] = lds(xa[u] + uint32_t(c) * xs[u]);
                double pr[SR][BS];
#pragma unroll
                for (int u = 0; u < SR; ++u) {
#pragma unroll
                    for (int r = 0; r < BS; ++r) pr[u][r] = vblk(u, r) * x[u][0];
#pragma unroll
                    for (int c = 1; c < BS; ++c)
#pragma unroll
                        for (int r = 0; r < BS; ++r) pr[u][r] = fma(vblk(u, c * BS + r), x[u][c], pr[u][r]);
                }
#pragma unroll
                for (int w = 1; w < SR; w <<= 1)
#pragma unroll
                    for (int u = 0; u + w < SR; u += 2 * w)
#pragma unroll
                        for (int r = 0; r < BS; ++r) pr[u][r] += pr[u + w][r];
#pragma unroll
                for (int r = 0; r < BS; ++r) acc[r] -= pr[0][r];
                smem_slots(gt, SR, acc);
                if (dbg) dbg[4] = clock64();
                publish(gt, idx, acc);
                if (dbg) dbg[5] = clock64();
            }
            // hand record i+1 to the next group, release record i's ring space
            if (i + 1 < nrec) named_bar_arrive(1 + (grp + 1) % G, 2 * PS_NG);
            if (dbg) dbg[6] = clock64();
            mbar_arrive(empty_bar + s);
            if (dbg) dbg[7] = clock64();
            if (a.trace && gt == 0) {
                a.trace[size_t(r0 + i) * 8 + 5] = globaltimer();
                uint32_t smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                a.trace[size_t(r0 + i) * 8 + 6] = (uint64_t(blockIdx.x) << 32) | smid;
                a.trace[size_t(r0 + i) * 8 + 7] = uint64_t(uint32_t(h.flags));
            }
        }
        if (!ldone) arrive_ldone();
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

// b in L-position order (the L records' input bulk copies read it)
template <int BS>
__global__ void permute_b_kernel(int64_t n, const int32_t *__restrict__ lrow, const double *__restrict__ b,
                                 double *__restrict__ bp, const int *skip) {
    if (skip && ld_relaxed_s32(skip) != 0) return;
    // a gather: position p takes b's row lrow[p]; the packed writes (the
    // costlier side of a permutation) are coalesced.  U positions per thread
    // and step, their loads issued together (the reads are scattered rows:
    // latency-bound without several in flight)
    constexpr int U = 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t p0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p0 < n; p0 += stride * U) {
        int64_t rows[U];
#pragma unroll
        for (int u = 0; u < U; ++u) rows[u] = p0 + u * stride < n ? __ldg(lrow + p0 + u * stride) : -1;
        double v[U][BS];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < BS; ++c) v[u][c] = rows[u] >= 0 ? __ldg(b + rows[u] * BS + c) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (rows[u] >= 0) {
                double *d = bp + size_t(p0 + u * stride) * BS;
#pragma unroll
                for (int c = 0; c < BS; ++c) d[c] = v[u][c];
            }
    }
}

// ===========================================================================
// pack: scatter the index sections and fill the value areas of every record
// from the factored P' values (L blocks verbatim, U' = D^-1 U after the split)
// and D^-1; one warp per record.
// ===========================================================================
template <int BS>
__global__ void ppack_kernel(int64_t nrec, const PRecInfo *__restrict__ info, const int32_t *__restrict__ idx,
                             const int32_t *__restrict__ vmap, unsigned char *__restrict__ recs,
                             const double *__restrict__ pvals, const double *__restrict__ dinv) {
    constexpr int BS2 = BS * BS;
    const int lane = threadIdx.x & 31;
    const int64_t W = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nrec; r += W) {
        const PRecInfo ri = info[r];
        int32_t *dst = reinterpret_cast<int32_t *>(recs + ri.off);
        const int32_t *src = idx + ri.idx_off;
        for (uint32_t w = lane; w < ri.idx_words; w += 32) dst[w] = src[w];
        const PRecHdr h = *reinterpret_cast<const PRecHdr *>(src);
        const int nr = ri.nrows;
        double *vals = reinterpret_cast<double *>(recs + ri.off + h.vals_off);
        if ((h.flags & 1)) {
            const int32_t *rows = src + sizeof(PRecHdr) / 4;
            for (int e = lane; e < BS2 * nr; e += 32) {
                const int el = e / nr, q = e - el * nr;
                vals[e] = dinv[int64_t(uint32_t(rows[q]) & ~PS_PUB) * BS2 + el];
            }
            vals += int64_t(BS2) * nr;
        }
        const int64_t tot = int64_t(ri.S) * BS2 * nr;
        for (int64_t e = lane; e < tot; e += 32) {
            const int64_t sl = e / (int64_t(BS2) * nr);
            const int rem = int(e - sl * BS2 * nr);
            const int el = rem / nr, q = rem - el * nr;
            const int32_t slot = vmap[ri.vmap_off + sl * nr + q];
            vals[e] = slot >= 0 ? pvals[int64_t(slot) * BS2 + el] : 0.0;
        }
        // padding bytes between the index section and the values stay as
        // cudaMalloc left them: they are never read
    }
}

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

size_t psweep_smem_bytes(const Plan &p) {
    const PSweep &ps = p.ps;
    return size_t(align128(int64_t(ps.ring + 2) * ps_vec_stride(p.bs) * 8)) + size_t(ps.xval_ring) + size_t(ps.data_ring);
}

cudaError_t launch_ppack(const Plan &p, cudaStream_t s) {
    const PSweep &ps = p.ps;
    const int64_t nrec = int64_t(ps.rec.size());
    if (nrec == 0) return cudaSuccess;
    const PRecInfo *info = reinterpret_cast<const PRecInfo *>(p.ws + p.off.ps_info);
    const int32_t *idx = reinterpret_cast<const int32_t *>(p.ws + p.off.ps_idx);
    const int32_t *vmap = reinterpret_cast<const int32_t *>(p.ws + p.off.ps_vmap);
    unsigned char *recs = p.ws + p.off.ps_rec;
    const double *pv = reinterpret_cast<const double *>(p.ws + p.off.pvals);
    const double *dv = reinterpret_cast<const double *>(p.ws + p.off.dinv);
    int64_t grid = (nrec + 7) / 8;
    if (grid > int64_t(p.num_sms) * 64) grid = int64_t(p.num_sms) * 64;
#define PPACK_LAUNCH(BS) ppack_kernel<BS><<<unsigned(grid), 256, 0, s>>>(nrec, info, idx, vmap, recs, pv, dv);
    BILUK_BS_DISPATCH(p.bs, PPACK_LAUNCH)
#undef PPACK_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_permute_b(const Plan &p, const double *b, cudaStream_t s, const int *skip) {
    const int32_t *posl = reinterpret_cast<const int32_t *>(p.ws + p.off.ps_posl);
    double *bp = reinterpret_cast<double *>(p.ws + p.off.ps_bperm);
    int64_t grid = (p.n + 255) / 256;
    if (grid > int64_t(p.num_sms) * 16) grid = int64_t(p.num_sms) * 16;
    if (grid < 1) grid = 1;
#define PERM_LAUNCH(BS) permute_b_kernel<BS><<<unsigned(grid), 256, 0, s>>>(p.n, posl, b, bp, skip);
    BILUK_BS_DISPATCH(p.bs, PERM_LAUNCH)
#undef PERM_LAUNCH
    return cudaGetLastError();
}

// the kernel instantiation of a plan: compute groups x producer warps
template <int BS>
static const void *psweep_fn(int groups, int nprod) {
    if (groups == 2)
        return nprod == 1 ? reinterpret_cast<const void *>(psweep_kernel<BS, 2, 1>)
                          : reinterpret_cast<const void *>(psweep_kernel<BS, 2, 2>);
    if (nprod == 4 && BS <= 4) return reinterpret_cast<const void *>(psweep_kernel<BS, 3, 4>);
    if (nprod == 3 && BS <= 4) return reinterpret_cast<const void *>(psweep_kernel<BS, 3, 3>);
    return nprod == 1 ? reinterpret_cast<const void *>(psweep_kernel<BS, 3, 1>)
                      : reinterpret_cast<const void *>(psweep_kernel<BS, 3, 2>);
}

static cudaError_t psweep_kernel_of(const Plan &p, const void **fn) {
#define PSWEEP_FN(BS) *fn = psweep_fn<BS>(p.ps.groups, p.ps.nprod);
    BILUK_BS_DISPATCH(p.bs, PSWEEP_FN)
#undef PSWEEP_FN
    return cudaSuccess;
}

static int psweep_threads(const Plan &p) { return p.ps.groups * PS_NG + 32 * p.ps.nprod; }

cudaError_t launch_psweep(const Plan &p, const PSweepArgs &a, cudaStream_t s) {
    const size_t smem = psweep_smem_bytes(p);
    const void *fn = nullptr;
    cudaError_t e = psweep_kernel_of(p, &fn);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    void *args[] = {const_cast<PSweepArgs *>(&a)};
    e = cudaLaunchCooperativeKernel(fn, dim3(p.ps.P), dim3(psweep_threads(p)), args, smem, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t psweep_occupancy(const Plan &p, int *blocks_per_sm) {
    const size_t smem = psweep_smem_bytes(p);
    const void *fn = nullptr;
    cudaError_t e = psweep_kernel_of(p, &fn);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, psweep_threads(p), smem);
}

}  // namespace biluk
