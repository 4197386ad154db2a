// bubble.cu — the polling synchronizer of rollout pre-generation (P:176-181:
// "during the pre-generation of B_{t+1}, each rank queries a central synchronizer every T
// decoding steps.  If the synchronizer reports that all ranks have completed B_t,
// pre-generation is halted"; T = 50 in the paper's setup).
//
// The synchronizer is a small array of per-rank words, hosted in the owner rank's HBM and
// mapped into every other rank's address space over NVLink (CUDA IPC).  A rank that finished
// B_t stores rl_step into its own word (system-scope release store, one 8-byte NVLink write);
// a poll is one kernel that reads the `world` words (system-scope acquire loads) and writes a
// halt flag in the caller's device memory.  Both are stream-ordered kernels, so a chunk of T
// pre-generation steps plus its poll is one CUDA graph replay: no collective (a slow rank never
// waits on a fast one), no host round trip inside the chunk.  Words are monotone (the latest
// finished rl_step), so nothing is reset between RL steps.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <new>
#include <string>

#include "../../include/bubblespec.h"
#include "common.cuh"

struct bs_bubble_sync {
    int device = 0;
    int owner = 0;                        // allocated here (freed on destroy) vs opened via IPC
    unsigned long long* words = nullptr;  // [BS_BUBBLE_MAX_RANKS]
    std::string err;
};

namespace bs {

__global__ void bubble_arrive_kernel(unsigned long long* words, int rank, unsigned long long step) {
    // the rank's batch is complete on this stream: publish it to every poller (system scope:
    // the word may live in a peer GPU's memory)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(words + rank), "l"(step) : "memory");
}

__global__ void bubble_poll_kernel(const unsigned long long* words, int world, unsigned long long step,
                                   int32_t* halt) {
    const int lane = threadIdx.x;
    bool done = true;
    for (int r = lane; r < world; r += 32) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(words + r) : "memory");
        done = done && (v != ~0ull) && v >= step;
    }
    done = __all_sync(0xFFFFFFFFu, done);
    if (lane == 0) *halt = done ? 1 : 0;
}

}  // namespace bs

static bs_status sync_fail(bs_bubble_sync* s, bs_status st, const char* what) {
    if (s) s->err = what;
    return st;
}

extern "C" {

bs_status bs_bubble_sync_create(int32_t device, bs_bubble_sync** out) {
    if (!out) return BS_ERR_INVALID;
    *out = nullptr;
    bs::DeviceScope dev_scope_(device);
    if (dev_scope_.err != cudaSuccess) return BS_ERR_CUDA;
    auto* s = new (std::nothrow) bs_bubble_sync();
    if (!s) return BS_ERR_OOM;
    s->device = device;
    s->owner = 1;
    if (cudaMalloc(&s->words, sizeof(unsigned long long) * BS_BUBBLE_MAX_RANKS) != cudaSuccess) {
        delete s;
        return BS_ERR_OOM;
    }
    // ~0: no RL step finished yet
    if (cudaMemset(s->words, 0xFF, sizeof(unsigned long long) * BS_BUBBLE_MAX_RANKS) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        cudaFree(s->words);
        delete s;
        return BS_ERR_CUDA;
    }
    *out = s;
    return BS_OK;
}

bs_status bs_bubble_sync_export(const bs_bubble_sync* s, void* handle64) {
    if (!s || !handle64 || !s->owner) return BS_ERR_INVALID;
    bs::DeviceScope dev_scope_(s->device);
    if (dev_scope_.err != cudaSuccess) return BS_ERR_CUDA;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, s->words) != cudaSuccess) return BS_ERR_CUDA;
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle64, &h, sizeof h);
    return BS_OK;
}

bs_status bs_bubble_sync_open(int32_t device, const void* handle64, bs_bubble_sync** out) {
    if (!out || !handle64) return BS_ERR_INVALID;
    *out = nullptr;
    bs::DeviceScope dev_scope_(device);
    if (dev_scope_.err != cudaSuccess) return BS_ERR_CUDA;
    auto* s = new (std::nothrow) bs_bubble_sync();
    if (!s) return BS_ERR_OOM;
    s->device = device;
    s->owner = 0;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof h);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        delete s;
        return BS_ERR_CUDA;
    }
    s->words = static_cast<unsigned long long*>(p);
    *out = s;
    return BS_OK;
}

void bs_bubble_sync_destroy(bs_bubble_sync* s) {
    if (!s) return;
    bs::DeviceScope dev_scope_(s->device);
    if (s->owner) cudaFree(s->words);
    else cudaIpcCloseMemHandle(s->words);
    delete s;
}

bs_status bs_bubble_sync_arrive(bs_bubble_sync* s, int32_t rank, uint64_t rl_step, void* stream) {
    if (!s || rank < 0 || rank >= BS_BUBBLE_MAX_RANKS || rl_step == ~0ull) return BS_ERR_INVALID;
    bs::DeviceScope dev_scope_(s->device);
    if (dev_scope_.err != cudaSuccess) return BS_ERR_CUDA;
    // a plain (fully stream-ordered) launch: the rank's last decoding step has completed
    bs::bubble_arrive_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(s->words, (int)rank,
                                                                              (unsigned long long)rl_step);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BS_OK : sync_fail(s, BS_ERR_CUDA, cudaGetErrorString(e));
}

bs_status bs_bubble_sync_poll(bs_bubble_sync* s, int32_t world, uint64_t rl_step, int32_t* halt,
                              void* stream) {
    if (!s || !halt || world < 1 || world > BS_BUBBLE_MAX_RANKS) return BS_ERR_INVALID;
    bs::DeviceScope dev_scope_(s->device);
    if (dev_scope_.err != cudaSuccess) return BS_ERR_CUDA;
    bs::bubble_poll_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        (const unsigned long long*)s->words, (int)world, (unsigned long long)rl_step, halt);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BS_OK : sync_fail(s, BS_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
