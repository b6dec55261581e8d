// Small sm_100a device helpers: memory-model-correct relaxed loads/stores for
// the sync-free sweeps, parity tags, mbarrier + bulk async copy (TMA 1-D).
#pragma once

#include <cstdint>

#include "biluk_internal.h"

namespace biluk {
namespace dev {

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- relaxed gpu-scope accesses (LDG/STG .STRONG.GPU: bypass L1, coherent at L2)
__device__ __forceinline__ double ld_relaxed(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_s32(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---- vector relaxed accesses (up to 256-bit, sm_100a LDG/STG.E.256.STRONG.GPU)
__device__ __forceinline__ void ld_relaxed_v2(const double *p, double &a, double &b) {
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld_relaxed_v4(const double *p, double &a, double &b, double &c, double &d) {
    asm volatile("ld.relaxed.gpu.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ void st_relaxed_v2(double *p, double a, double b) {
    asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void st_relaxed_v4(double *p, double a, double b, double c, double d) {
    asm volatile("st.relaxed.gpu.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
                 : "memory");
}
// a block row of the sweep vectors: BS values at p (stride vec_stride(BS), aligned),
// moved with the fewest vector instructions (4 / 2 / 1 doubles)
template <int BS>
__device__ __forceinline__ void ld_row(const double *p, double (&v)[BS]) {
    constexpr int N4 = BS / 4, O2 = 4 * N4, H2 = (BS - O2) / 2, O1 = O2 + 2 * H2, H1 = BS - O1;
#pragma unroll
    for (int k = 0; k < N4; ++k) ld_relaxed_v4(p + 4 * k, v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    if constexpr (H2 > 0) ld_relaxed_v2(p + O2, v[O2], v[O2 + 1]);
    if constexpr (H1 > 0) v[O1] = ld_relaxed(p + O1);
}
template <int BS>
__device__ __forceinline__ void st_row(double *p, const double (&v)[BS]) {
    if constexpr (BS == 3) {   // pad the 4th double: one 256-bit store
        st_relaxed_v4(p, v[0], v[1], v[2], 0.0);
    } else {
        constexpr int N4 = BS / 4, O2 = 4 * N4, H2 = (BS - O2) / 2, O1 = O2 + 2 * H2, H1 = BS - O1;
#pragma unroll
        for (int k = 0; k < N4; ++k) st_relaxed_v4(p + 4 * k, v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        if constexpr (H2 > 0) st_relaxed_v2(p + O2, v[O2], v[O2 + 1]);
        if constexpr (H1 > 0) st_relaxed(p + O1, v[O1]);
    }
}

// ---- parity tags.  Every word a sweep publishes carries the apply epoch's
// parity in its LSB.  A consumer polls the words themselves: each is its own
// ready flag, so a dependency costs ONE L2 round trip and no fences; no reset
// pass is needed because every row is rewritten exactly once per apply and the
// parity alternates.  A TAGGED ROW is exact: words 0..BS-1 hold the values with
// their LSB replaced by the tag, word BS holds the BS displaced LSBs (bits
// 1..BS) and the tag (bit 0); tag_stride(BS) >= BS + 1 words per row.
__device__ __forceinline__ uint32_t tag_of(double v) {
    return static_cast<uint32_t>(__double_as_longlong(v)) & 1u;
}
__device__ __forceinline__ double bits_as_double(unsigned long long b) {
    return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ unsigned long long double_bits(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v));
}
// the BS + 1 tagged words of a row
template <int BS>
__device__ __forceinline__ void tag_row(const double (&v)[BS], uint32_t par, double (&w)[BS + 1]) {
    unsigned long long lsb = par;
#pragma unroll
    for (int c = 0; c < BS; ++c) {
        const unsigned long long b = double_bits(v[c]);
        lsb |= (b & 1ull) << (c + 1);
        w[c] = bits_as_double((b & ~1ull) | par);
    }
    w[BS] = bits_as_double(lsb);
}
template <int BS>
__device__ __forceinline__ bool row_ready(const double (&w)[BS + 1], uint32_t par) {
    uint32_t ok = 1;
#pragma unroll
    for (int c = 0; c <= BS; ++c) ok &= (tag_of(w[c]) == par);
    return ok != 0;
}
// the exact values of a ready row
template <int BS>
__device__ __forceinline__ void untag_row(const double (&w)[BS + 1], double (&v)[BS]) {
    const unsigned long long lsb = double_bits(w[BS]);
#pragma unroll
    for (int c = 0; c < BS; ++c) v[c] = bits_as_double((double_bits(w[c]) & ~1ull) | ((lsb >> (c + 1)) & 1ull));
}
// N consecutive doubles at p (32-byte aligned when N >= 3, 16-byte when N == 2),
// relaxed gpu-scope, the fewest vector accesses; N = 3 is read/written as 4
// (the 4th word belongs to the same row's padding)
template <int N>
__device__ __forceinline__ void ld_words(const double *p, double (&w)[N]) {
    if constexpr (N == 4) {   // two 128-bit loads measured faster than one 256-bit load (tiled sweep 1118 vs 1246 us)
        ld_relaxed_v2(p, w[0], w[1]);
        ld_relaxed_v2(p + 2, w[2], w[3]);
        return;
    }
    constexpr int N4 = N / 4, R = N - 4 * N4;
#pragma unroll
    for (int k = 0; k < N4; ++k) ld_relaxed_v4(p + 4 * k, w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
    if constexpr (R == 3) {
        double d;
        ld_relaxed_v4(p + 4 * N4, w[4 * N4], w[4 * N4 + 1], w[4 * N4 + 2], d);
    } else if constexpr (R == 2) {
        ld_relaxed_v2(p + 4 * N4, w[4 * N4], w[4 * N4 + 1]);
    } else if constexpr (R == 1) {
        w[4 * N4] = ld_relaxed(p + 4 * N4);
    }
}
template <int N>
__device__ __forceinline__ void st_words(double *p, const double (&w)[N]) {
    constexpr int N4 = N / 4, R = N - 4 * N4;
#pragma unroll
    for (int k = 0; k < N4; ++k) st_relaxed_v4(p + 4 * k, w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
    if constexpr (R == 3) {
        st_relaxed_v4(p + 4 * N4, w[4 * N4], w[4 * N4 + 1], w[4 * N4 + 2], 0.0);
    } else if constexpr (R == 2) {
        st_relaxed_v2(p + 4 * N4, w[4 * N4], w[4 * N4 + 1]);
    } else if constexpr (R == 1) {
        st_relaxed(p + 4 * N4, w[4 * N4]);
    }
}
// publish / poll one tagged row (tag_stride(BS) doubles at p)
template <int BS>
__device__ __forceinline__ void st_tagged(double *p, const double (&v)[BS], uint32_t par) {
    double w[BS + 1];
    tag_row<BS>(v, par, w);
    st_words<BS + 1>(p, w);
}
template <int BS>
__device__ __forceinline__ void ld_tagged(const double *p, double (&w)[BS + 1]) {
    ld_words<BS + 1>(p, w);
}
// the same with the values landing in v and the LSB word in lw (no extra
// buffer: callers polling many rows keep one register set per row)
template <int BS>
__device__ __forceinline__ void ld_tagged_split(const double *p, double (&v)[BS], double &lw) {
    double w[BS + 1];
    ld_words<BS + 1>(p, w);
#pragma unroll
    for (int c = 0; c < BS; ++c) v[c] = w[c];
    lw = w[BS];
}
// restore exact values in place from a ready split row
template <int BS>
__device__ __forceinline__ void untag_split(double (&v)[BS], double lw) {
    const unsigned long long lsb = double_bits(lw);
#pragma unroll
    for (int c = 0; c < BS; ++c) v[c] = bits_as_double((double_bits(v[c]) & ~1ull) | ((lsb >> (c + 1)) & 1ull));
}

// ---- mbarrier + bulk async copy (cp.async.bulk, the 1-D TMA path)
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    while (!mbar_try_wait(bar, phase)) {
    }
}

// ===========================================================================
// small dense block inverse: LU with partial pivoting, the rules of
// block_invert (factor.py:38-70): all-zero block singular, |pivot| <
// 1e-13 * max|B| singular, first maximal pivot wins (np.argmax).
// a: column-major input (a[c*BS + r]); inv: column-major output.
// ===========================================================================
template <int BS>
__device__ __forceinline__ bool block_invert(const double *a, double *inv) {
    double lu[BS][BS];
    double amax = 0.0;
#pragma unroll
    for (int r = 0; r < BS; ++r)
#pragma unroll
        for (int c = 0; c < BS; ++c) {
            lu[r][c] = a[c * BS + r];
            amax = fmax(amax, fabs(lu[r][c]));
        }
    if (amax == 0.0) return false;
    if (BS == 1) {
        inv[0] = 1.0 / lu[0][0];
        return true;
    }
    int perm[BS];
#pragma unroll
    for (int r = 0; r < BS; ++r) perm[r] = r;
#pragma unroll
    for (int c = 0; c < BS; ++c) {
        int p = c;
        double best = fabs(lu[c][c]);
#pragma unroll
        for (int r = c + 1; r < BS; ++r)
            if (fabs(lu[r][c]) > best) {
                best = fabs(lu[r][c]);
                p = r;
            }
        if (best < 1e-13 * amax) return false;
        if (p != c) {
#pragma unroll
            for (int q = 0; q < BS; ++q) {
                const double t = lu[c][q];
                lu[c][q] = lu[p][q];
                lu[p][q] = t;
            }
            const int t = perm[c];
            perm[c] = perm[p];
            perm[p] = t;
        }
#pragma unroll
        for (int r = c + 1; r < BS; ++r) {
            lu[r][c] /= lu[c][c];
#pragma unroll
            for (int q = c + 1; q < BS; ++q) lu[r][q] -= lu[r][c] * lu[c][q];
        }
    }
    // X = U^-1 L^-1 P  (row r of P is e_{perm[r]})
    double x[BS][BS];
#pragma unroll
    for (int r = 0; r < BS; ++r)
#pragma unroll
        for (int q = 0; q < BS; ++q) x[r][q] = (perm[r] == q) ? 1.0 : 0.0;
#pragma unroll
    for (int r = 1; r < BS; ++r)
#pragma unroll
        for (int q = 0; q < BS; ++q) {
            double s = 0.0;
#pragma unroll
            for (int m = 0; m < r; ++m) s += lu[r][m] * x[m][q];
            x[r][q] -= s;
        }
#pragma unroll
    for (int r = BS - 1; r >= 0; --r)
#pragma unroll
        for (int q = 0; q < BS; ++q) {
            double s = 0.0;
#pragma unroll
            for (int m = r + 1; m < BS; ++m) s += lu[r][m] * x[m][q];
            x[r][q] = (x[r][q] - s) / lu[r][r];
        }
#pragma unroll
    for (int r = 0; r < BS; ++r)
#pragma unroll
        for (int q = 0; q < BS; ++q) inv[q * BS + r] = x[r][q];
    return true;
}

}  // namespace dev
}  // namespace biluk
