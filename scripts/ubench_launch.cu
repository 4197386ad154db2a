// Fixed cost of launching the verify kernel's grid shape: an (almost) empty kernel with
// 8-CTA clusters, 384 threads and 83 KB dynamic smem per CTA, for several grid sizes,
// replayed back to back from a CUDA graph (per-launch device time).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubl scripts/ubench_launch.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(384, 2) k_cluster(int* o) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] < 0) o[0] = 1;
}
__global__ void __launch_bounds__(384, 2) k_plain(int* o) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] < 0) o[0] = 1;
}
int main() {
    int* o;
    cudaMalloc(&o, 4);
    const int smem = 83 * 1024;
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int kind = 0; kind < 2; ++kind)
        for (int grid : {8, 72, 264}) {
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < 64; ++i) {
                if (kind == 0) k_cluster<<<grid, 384, smem, st>>>(o);
                else k_plain<<<grid, 384, smem, st>>>(o);
            }
            cudaStreamEndCapture(st, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, st);
            cudaStreamSynchronize(st);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, st);
            cudaGraphLaunch(ge, st);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%s grid %3d: %.2f us per launch\n", kind ? "plain  " : "cluster", grid, ms * 1e3 / 64);
        }
    return 0;
}
