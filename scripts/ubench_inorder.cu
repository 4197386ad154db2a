// Does a shared-memory op issued after an outstanding global atomic / load wait for it?
// (the verify claimer's loop showed a ~1.2 us ATOMS right after a pre-issued claim atomic)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubi scripts/ubench_inorder.cu && /tmp/ubi
#include <cstdio>
#include <cuda_runtime.h>
// mode bit0: a global atomic first; bit1: an L2 load first; bit2: probe an mbarrier instead of ATOMS;
// bit3: probe with a plain LDS
__global__ void k(unsigned long long* g, const unsigned long long* h, long long* out, int mode) {
    __shared__ unsigned int s;
    __shared__ unsigned long long bar;
    if (threadIdx.x == 0) {
        s = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    }
    __syncthreads();
    unsigned long long v = 0;
    long long t0 = clock64();
    if (mode & 1) v = atomicAdd(g + 64 * blockIdx.x, 1ull);
    if (mode & 2) v += __ldcg(h + 4096 * blockIdx.x);
    unsigned x;
    if (mode & 4) {
        unsigned ok;
        asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
        x = ok;
    } else if (mode & 8) {
        x = *(volatile unsigned*)&s;
    } else {
        x = atomicOr(&s, 0u);
    }
    x = __shfl_sync(0xFFFFFFFFu, x, 0);  // waits for x
    long long t1 = clock64();
    unsigned long long w = __shfl_sync(0xFFFFFFFFu, v, 0);  // waits for the global op
    long long t2 = clock64();
    out[blockIdx.x * 4 + 0] = t1 - t0;
    out[blockIdx.x * 4 + 1] = t2 - t0;
    out[blockIdx.x * 4 + 3] = (long long)(w + x);
}
int main() {
    unsigned long long *g, *h;
    long long* o;
    cudaMalloc(&g, 1 << 26);
    cudaMalloc(&h, 1 << 28);
    cudaMemset(g, 0, 1 << 26);
    cudaMemset(h, 0, 1 << 28);
    cudaMallocManaged(&o, 1024 * 32);
    int modes[] = {0, 1, 2, 4, 5, 6, 8, 9, 10};
    for (int mode : modes) {
        for (int rep = 0; rep < 3; ++rep) {
            k<<<1, 32>>>(g, h, o, mode);
            cudaDeviceSynchronize();
        }
        printf("mode %2d (%s%s %s): smem result after %lld cycles, global result after %lld\n", mode,
               mode & 1 ? "atomicAdd(global) " : "", mode & 2 ? "ldcg " : "",
               mode & 4 ? "then mbarrier.test_wait" : (mode & 8 ? "then LDS" : "then ATOMS"), o[0], o[1]);
    }
    return 0;
}
