// The reference's sub-stage entry points as device operations (the drop-in
// surface of blockiluk/__init__.py:51-86 beyond build / apply / gmres):
//   block_invert (factor.py:38-70)          -> biluk_block_invert (batched)
//   apply_block_diagonal (trisolve.py:148)  -> biluk_block_diag_apply
//   materialize (factor.py:83-121)          -> biluk_scatter_blocks (the host computes the slot map)
//   block/point_ilu0_factorize (:151-205)   -> biluk_plan_factor_lu (no split)
//   split_ldu (factor.py:230-289)           -> biluk_plan_load_factored (D^-1 of the
//                                              diagonal blocks, U' = D^-1 U, sweep records)
// solve_unit_triangular (trisolve.py:121-145) runs the sweep of a plan loaded
// with (I + T) as its factored matrix (unit D, T as L or U').
#include <cuda_runtime.h>

#include <string>

#include "biluk_internal.h"
#include "device_util.cuh"
#include "kernels.cuh"

namespace biluk {

using namespace dev;

namespace {

#define STAGE_BS_DISPATCH(bs, F)  \
    switch (bs) {                 \
        case 1: F(1); break;      \
        case 2: F(2); break;      \
        case 3: F(3); break;      \
        case 4: F(4); break;      \
        case 5: F(5); break;      \
        case 6: F(6); break;      \
        case 7: F(7); break;      \
        case 8: F(8); break;      \
        default: return fail(BILUK_EUNSUPPORTED, "block size must be in 1..8"); \
    }

unsigned grid_of(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    if (g > 148 * 64) g = 148 * 64;
    return unsigned(g < 1 ? 1 : g);
}

// inverses of n row-major blocks (the reference's (n, bs, bs) layout); the
// first singular block index is atomicMin'ed into *bad
template <int BS>
__global__ void block_invert_kernel(int64_t n, const double *__restrict__ in, double *__restrict__ out,
                                    unsigned long long *bad) {
    constexpr int BS2 = BS * BS;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        double a[BS2], inv[BS2];
        // row-major (r, c) at in[r*BS + c] is column-major element c*BS + r of the transpose:
        // read it transposed into column-major order
#pragma unroll
        for (int r = 0; r < BS; ++r)
#pragma unroll
            for (int c = 0; c < BS; ++c) a[c * BS + r] = in[i * BS2 + r * BS + c];
        const bool ok = block_invert<BS>(a, inv);
#pragma unroll
        for (int r = 0; r < BS; ++r)
#pragma unroll
            for (int c = 0; c < BS; ++c) out[i * BS2 + r * BS + c] = ok ? inv[c * BS + r] : 0.0;
        if (!ok) atomicMin(bad, (unsigned long long)i);
    }
}

// z_I = dinv[I] @ y_I, dinv row-major (n, bs, bs)
template <int BS>
__global__ void block_diag_kernel(int64_t n, const double *__restrict__ dinv, const double *__restrict__ y,
                                  double *__restrict__ z) {
    constexpr int BS2 = BS * BS;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        double yv[BS];
#pragma unroll
        for (int c = 0; c < BS; ++c) yv[c] = y[i * BS + c];
#pragma unroll
        for (int r = 0; r < BS; ++r) {
            double s = dinv[i * BS2 + r * BS] * yv[0];
#pragma unroll
            for (int c = 1; c < BS; ++c) s = fma(dinv[i * BS2 + r * BS + c], yv[c], s);
            z[i * BS + r] = s;
        }
    }
}

__global__ void scatter_blocks_kernel(int64_t nsrc, int bs2, const int64_t *__restrict__ map,
                                      const double *__restrict__ src, double *__restrict__ dst) {
    const int64_t total = nsrc * bs2;
    for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s = g / bs2;
        dst[map[s] * bs2 + (g - s * bs2)] = src[g];
    }
}

// D_i^-1 of the diagonal blocks of a factored matrix held in the plan's value
// array (column-major blocks), the rules of block_invert; singular -> the
// plan's factorization status (first row by atomicMin)
template <int BS>
__global__ void diag_invert_kernel(int64_t n, const int32_t *__restrict__ diag, const double *__restrict__ pvals,
                                   double *__restrict__ dinv, DevStatus *st) {
    constexpr int BS2 = BS * BS;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        double inv[BS2];
        const bool ok = block_invert<BS>(pvals + int64_t(diag[i]) * BS2, inv);
#pragma unroll
        for (int x = 0; x < BS2; ++x) dinv[i * BS2 + x] = ok ? inv[x] : 0.0;
        if (!ok) {
            atomicExch(&st->fstatus, BILUK_ESINGULAR);
            atomicMin(&st->ferr_row, (long long)i);
        }
    }
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(BILUK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

cudaError_t launch_diag_invert(const Plan &p, cudaStream_t s) {
    const int32_t *dg = reinterpret_cast<const int32_t *>(p.ws + p.off.p_diag);
    const double *pv = reinterpret_cast<const double *>(p.ws + p.off.pvals);
    double *dv = reinterpret_cast<double *>(p.ws + p.off.dinv);
    DevStatus *st = reinterpret_cast<DevStatus *>(p.ws + p.off.status);
    if (p.n == 0) return cudaSuccess;
#define DINV_LAUNCH(BS) diag_invert_kernel<BS><<<grid_of(p.n, 128), 128, 0, s>>>(p.n, dg, pv, dv, st); break;
    switch (p.bs) {
        case 1: DINV_LAUNCH(1)
        case 2: DINV_LAUNCH(2)
        case 3: DINV_LAUNCH(3)
        case 4: DINV_LAUNCH(4)
        case 5: DINV_LAUNCH(5)
        case 6: DINV_LAUNCH(6)
        case 7: DINV_LAUNCH(7)
        case 8: DINV_LAUNCH(8)
        default: return cudaErrorInvalidValue;
    }
#undef DINV_LAUNCH
    return cudaGetLastError();
}

}  // namespace biluk

using namespace biluk;

extern "C" {

int biluk_block_invert(int32_t bs, int64_t n, const double *dev_in, double *dev_out, int64_t *err_idx, void *stream) {
    if (n < 0 || (n > 0 && (!dev_in || !dev_out))) return fail(BILUK_EARG, "bad block_invert arguments");
    if (err_idx) *err_idx = -1;
    if (n == 0) return BILUK_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long *bad = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&bad), sizeof(*bad), s);
    if (e != cudaSuccess) return cuda_fail(e, "block_invert");
    e = cudaMemsetAsync(bad, 0xff, sizeof(*bad), s);
    if (e != cudaSuccess) return cuda_fail(e, "block_invert");
#define INV_LAUNCH(BS) block_invert_kernel<BS><<<grid_of(n, 128), 128, 0, s>>>(n, dev_in, dev_out, bad);
    STAGE_BS_DISPATCH(bs, INV_LAUNCH)
#undef INV_LAUNCH
    unsigned long long h = ~0ull;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(bad, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "block_invert");
    if (h != ~0ull) {
        if (err_idx) *err_idx = int64_t(h);
        return fail(BILUK_ESINGULAR, "singular block " + std::to_string(h));
    }
    return BILUK_OK;
}

int biluk_block_diag_apply(int32_t bs, int64_t n, const double *dev_dinv, const double *dev_y, double *dev_z,
                           void *stream) {
    if (n < 0) return fail(BILUK_EARG, "negative dimension");
    if (n == 0) return BILUK_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
#define BD_LAUNCH(BS) block_diag_kernel<BS><<<grid_of(n, 128), 128, 0, s>>>(n, dev_dinv, dev_y, dev_z);
    STAGE_BS_DISPATCH(bs, BD_LAUNCH)
#undef BD_LAUNCH
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BILUK_OK : cuda_fail(e, "apply_block_diagonal");
}

int biluk_scatter_blocks(int32_t bs2, int64_t nsrc, const int64_t *dev_map, const double *dev_src, double *dev_dst,
                         void *stream) {
    if (nsrc < 0 || bs2 < 1) return fail(BILUK_EARG, "bad scatter arguments");
    if (nsrc == 0) return BILUK_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    scatter_blocks_kernel<<<grid_of(nsrc * bs2, 256), 256, 0, s>>>(nsrc, bs2, dev_map, dev_src, dev_dst);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BILUK_OK : cuda_fail(e, "materialize");
}

}  // extern "C"
