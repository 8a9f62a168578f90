// Grid-barrier cost probe (tools/ only): cooperative grid.sync() vs a flat
// atomic barrier vs a cluster-hierarchical one, 148 x k CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_probe gridsync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_cg(int n) {
    for (int i = 0; i < n; ++i) cg::this_grid().sync();
}

__global__ void k_flat(int n, unsigned* cnt) {
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
            const unsigned target = (unsigned)(i + 1) * gridDim.x;
            while (ld_acq(cnt) < target) {}
        }
        __syncthreads();
    }
}

__global__ void k_clu(int n, unsigned* cnt) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned ncl = gridDim.x / cl.num_blocks();
    for (int i = 0; i < n; ++i) {
        cl.sync();
        if (cl.block_rank() == 0 && threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
            const unsigned target = (unsigned)(i + 1) * ncl;
            while (ld_acq(cnt) < target) {}
        }
        cl.sync();
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* cnt;
    cudaMalloc(&cnt, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int n = 2000;
    for (int threads : {256, 896}) {
        for (int rep = 0; rep < 2; ++rep) {
            float ms;
            int nn = n;
            void* args[] = {&nn};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_cg, sms, threads, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("threads %d cg grid.sync: %.3f us\n", threads, ms * 1e3 / n);
            cudaMemset(cnt, 0, 4);
            void* args2[] = {&nn, &cnt};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_flat, sms, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("threads %d flat red/acquire: %.3f us\n", threads, ms * 1e3 / n);
            for (int cs : {2, 4, 8}) {
                if (sms % cs) continue;
                cudaMemset(cnt, 0, 4);
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(sms);
                cfg.blockDim = dim3(threads);
                cudaLaunchAttribute at[2];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                at[1].id = cudaLaunchAttributeCooperative;
                at[1].val.cooperative = 1;
                cfg.attrs = at;
                cfg.numAttrs = 2;
                cudaEventRecord(a);
                cudaError_t e = cudaLaunchKernelEx(&cfg, k_clu, nn, cnt);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                printf("threads %d cluster %d hierarchical: %.3f us (%s)\n", threads, cs, ms * 1e3 / n,
                       cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
