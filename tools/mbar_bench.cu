// Microbenchmark of the pipeline primitives on one SM (diagnostics):
// mbarrier try_wait / test_wait on a completed phase, arrive, and the issue
// cost + round trip of a 28 KB cp.async.bulk from global memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbar_bench tools/mbar_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool try_wait(uint64_t *b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ bool test_wait(uint64_t *b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t n, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                 "l"(src), "r"(n), "r"(sa(b)) : "memory");
}

__global__ void bench(const unsigned char *g, long long *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[4];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    arrive(bar + 0);   // phase 0 of bar[0] complete
    long long t0 = clock64();
    int acc = 0;
    for (int i = 0; i < 100; ++i) acc += try_wait(bar + 0, 0);
    long long t1 = clock64();
    for (int i = 0; i < 100; ++i) acc += test_wait(bar + 0, 0);
    long long t2 = clock64();
    for (int i = 0; i < 100; ++i) {   // arrive + wait cycle
        arrive(bar + 1);
        while (!try_wait(bar + 1, i & 1)) {
        }
    }
    long long t3 = clock64();
    // bulk copy: issue cost and round trip (28 KB, from L2 after the first)
    const uint32_t n = 28 * 1024;
    long long iss = 0, rt = 0;
    for (int i = 0; i < 20; ++i) {
        long long a = clock64();
        expect_tx(bar + 2, n);
        bulk(sm, g + (size_t(i) % 2) * n, n, bar + 2);
        long long b = clock64();
        while (!try_wait(bar + 2, i & 1)) {
        }
        long long c = clock64();
        if (i >= 4) {
            iss += b - a;
            rt += c - a;
        }
    }
    // two copies back to back (M + inputs)
    long long t4 = clock64();
    for (int i = 0; i < 16; ++i) {
        expect_tx(bar + 3, n + 4096);
        bulk(sm, g + (size_t(i) % 2) * n, n, bar + 3);
        bulk(sm + n, g + 3 * n, 4096, bar + 3);
        while (!try_wait(bar + 3, i & 1)) {
        }
    }
    long long t5 = clock64();
    out[0] = (t1 - t0) / 100;
    out[1] = (t2 - t1) / 100;
    out[2] = (t3 - t2) / 100;
    out[3] = iss / 16;
    out[4] = rt / 16;
    out[5] = (t5 - t4) / 16;
    out[6] = acc;
}

int main() {
    unsigned char *g;
    long long *o, h[8];
    cudaMalloc(&g, 4 << 20);
    cudaMemset(g, 1, 4 << 20);
    cudaMalloc(&o, 64);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    bench<<<1, 32, 64 * 1024>>>(g, o);
    cudaMemcpy(h, o, 64, cudaMemcpyDeviceToHost);
    printf("{\"try_wait_complete_cyc\": %lld, \"test_wait_complete_cyc\": %lld, \"arrive+wait_cyc\": %lld, "
           "\"bulk28k_issue_cyc\": %lld, \"bulk28k_roundtrip_cyc\": %lld, \"bulk28k+4k_roundtrip_cyc\": %lld, \"err\": \"%s\"}\n",
           h[0], h[1], h[2], h[3], h[4], h[5], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
