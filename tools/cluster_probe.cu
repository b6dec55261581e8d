// Feasibility probe: cooperative launch of 1-CTA-per-SM kernels (big shared
// memory) grouped in thread-block clusters; max active clusters; a DSMEM
// ping-pong latency between the two CTAs of a cluster.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_probe tools/cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__global__ void probe(unsigned long long *out, int iters) {
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cl = cg::this_cluster();
    volatile unsigned long long *flag = reinterpret_cast<unsigned long long *>(smem);
    if (threadIdx.x == 0) *flag = 0;
    cl.sync();
    const unsigned rank = cl.block_rank();
    volatile unsigned long long *peer = cl.map_shared_rank(const_cast<unsigned long long *>(flag), rank ^ 1u);
    unsigned long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0 && cl.num_blocks() >= 2 && rank < 2) {
        t0 = clock64();
        for (int i = 1; i <= iters; ++i) {
            if (rank == 0) {
                *peer = 2 * i - 1;                       // ping
                while (*flag != 2ull * i) {}             // wait for pong
            } else {
                while (*flag != 2ull * i - 1) {}
                *peer = 2 * i;
            }
        }
        t1 = clock64();
        if (rank == 0) out[blockIdx.x / cl.num_blocks()] = (t1 - t0) / iters;   // cycles per round trip
    }
    cl.sync();
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    unsigned long long *out;
    cudaMalloc(&out, 1024 * 8);
    for (int cs : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.blockDim = dim3(448);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        cfg.gridDim = dim3(cs);
        int maxc = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&maxc, probe, &cfg);
        int grid = (144 / cs) * cs;
        cfg.gridDim = dim3(grid);
        cudaError_t e2 = cudaLaunchKernelEx(&cfg, probe, out, 1000);
        cudaError_t e3 = cudaDeviceSynchronize();
        unsigned long long h[4] = {0, 0, 0, 0};
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        printf("cluster %d: max active clusters %d (%s) -> CTAs %d; launch grid %d: %s / %s; ping-pong %llu %llu cycles\n",
               cs, maxc, cudaGetErrorString(e), maxc * cs, grid, cudaGetErrorString(e2), cudaGetErrorString(e3), h[0], h[1]);
        cudaGetLastError();
    }
    return 0;
}
