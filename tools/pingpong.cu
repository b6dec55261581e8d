// Inter-SM flag ping-pong latency on the B200 (diagnostic microbenchmark).
// Two single-warp CTAs pass a counter back and forth through global memory;
// one hop = store by one SM -> observed by the poll of another SM.
// Optional background CTAs spin on private addresses to emulate polling load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pingpong tools/pingpong.cu && ./pingpong
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
template <int MODE>
__device__ __forceinline__ unsigned long long ld(const unsigned long long *p) {
    unsigned long long v;
    if (MODE == 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (MODE == 1) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (MODE == 2) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("atom.relaxed.gpu.global.or.b64 %0, [%1], 0;" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <int MODE>
__device__ __forceinline__ void st(unsigned long long *p, unsigned long long v) {
    if (MODE == 2) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else if (MODE == 1) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MODE>
__global__ void pingpong(unsigned long long *a, unsigned long long *b, int iters, unsigned long long *out,
                         volatile int *stop, unsigned long long *bg) {
    if (blockIdx.x >= 2) {   // background pollers
        unsigned long long *p = bg + blockIdx.x * 64 + (threadIdx.x & 31) * 2;
        while (*stop == 0) {
            unsigned long long v = ld<0>(p);
            if (v == 12345) st<0>(p + 1, v);
        }
        return;
    }
    if (threadIdx.x != 0) return;
    uint64_t t0 = gt();
    if (blockIdx.x == 0) {
        for (int k = 1; k <= iters; ++k) {
            st<MODE>(a, (unsigned long long)k);
            while (ld<MODE>(b) != (unsigned long long)k) {
            }
        }
        out[0] = gt() - t0;
        *stop = 1;
    } else {
        for (int k = 1; k <= iters; ++k) {
            while (ld<MODE>(a) != (unsigned long long)k) {
            }
            st<MODE>(b, (unsigned long long)k);
        }
    }
}

// sweep-like hop: a full warp polls NL loads per lane (component-major
// positions, like y_t), all lanes must see the token before publishing 3
// tagged doubles per lane; the partner warp does the same on other addresses.
template <int NL>
__global__ void warp_pingpong(double *va, double *vb, int64_t npos, int iters, unsigned long long *out) {
    if (blockIdx.x >= 2) return;
    const int lane = threadIdx.x;
    uint64_t t0 = gt();
    double *mine = blockIdx.x == 0 ? va : vb;
    double *other = blockIdx.x == 0 ? vb : va;
    for (int k = 1; k <= iters; ++k) {
        if (blockIdx.x == 0 || k > 0) {
            if (blockIdx.x == 0) {
                for (int c = 0; c < 3; ++c) {
                    double v = double(k);
                    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(mine + c * npos + lane), "d"(v) : "memory");
                }
            }
            // poll: NL loads per lane, the first 3 are the partner's components
            while (true) {
                double x[NL];
#pragma unroll
                for (int q = 0; q < NL; ++q) {
                    const double *p = other + (q % 3) * npos + lane + (q / 3) * 64;
                    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(x[q]) : "l"(p) : "memory");
                }
                bool ok = true;
#pragma unroll
                for (int q = 0; q < 3; ++q) ok &= (x[q] == double(k));
                if (__all_sync(0xffffffffu, ok)) break;
            }
            if (blockIdx.x == 1) {
                for (int c = 0; c < 3; ++c) {
                    double v = double(k);
                    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(mine + c * npos + lane), "d"(v) : "memory");
                }
            }
        }
    }
    if (blockIdx.x == 0 && lane == 0) out[0] = gt() - t0;
}

__global__ void dfma_latency(double *io, unsigned long long *out) {
    __shared__ double sm[256];
    sm[threadIdx.x] = io[threadIdx.x];
    __syncthreads();
    double a = io[0], b = io[1], c = io[2];
    long long c0 = clock64();
    for (int i = 0; i < 1000; ++i) a = fma(a, b, c);   // dependent chain
    long long c1 = clock64();
    double s = 0.0;
    int idx = threadIdx.x;
    for (int i = 0; i < 1000; ++i) {                     // dependent LDS chain
        s += sm[idx];
        idx = (idx + int(sm[idx] != 12345.0)) & 255;
    }
    long long c2 = clock64();
    float f = float(b), g = float(c), h = float(a);
    for (int i = 0; i < 1000; ++i) h = fmaf(h, f, g);
    long long c3 = clock64();
    io[8] = a + s + h;
    out[0] = c1 - c0;
    out[1] = c2 - c1;
    out[2] = c3 - c2;
}

__global__ void timer_cost(unsigned long long *out) {
    long long c0 = clock64();
    uint64_t acc = 0;
    for (int i = 0; i < 1000; ++i) acc += gt();
    long long c1 = clock64();
    for (int i = 0; i < 1000; ++i) acc += (uint64_t)clock64();
    long long c2 = clock64();
    out[0] = c1 - c0;
    out[1] = c2 - c1;
    out[2] = acc;
}

template <int NL>
void run_warp(const char *name) {
    double *buf;
    unsigned long long *out;
    const int64_t npos = 1 << 16;
    cudaMalloc(&buf, sizeof(double) * npos * 8);
    cudaMalloc(&out, 64);
    cudaMemset(buf, 0, sizeof(double) * npos * 8);
    const int iters = 2000;
    warp_pingpong<NL><<<2, 32>>>(buf, buf + npos * 4, npos, iters, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long ns = 0;
    cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"%s\", \"hop_ns\": %.1f, \"err\": \"%s\"}\n", name, double(ns) / (2.0 * iters),
           cudaGetErrorString(e));
    cudaFree(buf);
    cudaFree(out);
}

template <int MODE>
void run(const char *name, int bg_ctas, int far) {
    unsigned long long *buf, *out, *bgbuf;
    int *stop;
    cudaMalloc(&buf, 1 << 20);
    cudaMalloc(&out, 64);
    cudaMalloc(&stop, 4);
    cudaMalloc(&bgbuf, size_t(1 << 20) * 8);
    cudaMemset(buf, 0, 1 << 20);
    cudaMemset(stop, 0, 4);
    cudaMemset(bgbuf, 0, size_t(1 << 20) * 8);
    const int iters = 2000;
    unsigned long long *a = buf, *b = buf + (far ? 4096 : 16);
    pingpong<MODE><<<2 + bg_ctas, 32 * (bg_ctas ? 8 : 1)>>>(a, b, iters, out, stop, bgbuf);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long ns = 0;
    cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"%s\", \"bg_ctas\": %d, \"far\": %d, \"hop_ns\": %.1f, \"err\": \"%s\"}\n", name, bg_ctas, far,
           double(ns) / (2.0 * iters), cudaGetErrorString(e));
    cudaFree(buf);
    cudaFree(out);
    cudaFree(stop);
    cudaFree(bgbuf);
}

int main() {
    {
        unsigned long long *o, h[3];
        cudaMalloc(&o, 64);
        timer_cost<<<1, 1>>>(o);
        cudaMemcpy(h, o, 24, cudaMemcpyDeviceToHost);
        printf("{\"globaltimer_cycles_per_read\": %.1f, \"clock64_cycles_per_read\": %.1f}\n", h[0] / 1000.0,
               h[1] / 1000.0);
        double *io;
        cudaMalloc(&io, 4096);
        cudaMemset(io, 0, 4096);
        dfma_latency<<<1, 32>>>(io, o);
        cudaMemcpy(h, o, 24, cudaMemcpyDeviceToHost);
        printf("{\"dfma_dep_latency_cycles\": %.1f, \"lds_chain_cycles\": %.1f, \"ffma_dep_latency_cycles\": %.1f}\n",
               h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0);
        cudaFree(io);
        cudaFree(o);
    }
    for (int bg : {0, 146}) {
        run<0>("relaxed.gpu", bg, 1);
        run<1>("volatile", bg, 1);
        run<2>("acquire/release", bg, 1);
        run<3>("atom.or poll", bg, 1);
    }
    run<0>("relaxed.gpu same-line", 0, 0);
    run_warp<3>("warp 32 lanes x 3 loads (one dep, 3 components)");
    run_warp<9>("warp 32 lanes x 9 loads (3 deps)");
    run_warp<21>("warp 32 lanes x 21 loads (7 deps)");
    return 0;
}
