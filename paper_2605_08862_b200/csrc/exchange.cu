// exchange.cu — cross-rank draft exchange (K6, per RL step; "each rollout DP rank
// builds and maintains suffix indices only for the prompts it is responsible for"
// "dispatch pre-generated draft responses to each rollout rank according to their
// assigned prompts").  Drafts produced in any rank's bubble are all-gathered over NCCL
// (NVLink / NVSwitch) and each rank keeps the sequences of the prompts it owns
// (owner(P) = P mod R: round-robin dispatch by prompt).
//
// NCCL is loaded lazily with dlopen (libnccl.so.2: torch's bundled copy if already loaded,
// else the system one), so the library loads on machines without NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "ctx.h"

using namespace bs;

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
        api.AllGather = (decltype(api.AllGather))dlsym(api.h, "ncclAllGather");
        api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
                 api.GroupStart && api.GroupEnd;
    });
    return api;
}

__global__ void gather_seqs_kernel(int nkeep, const int64_t* src, const int64_t* dst,
                                   const int64_t* len, const int32_t* from, int32_t* to) {
    for (int s = blockIdx.x; s < nkeep; s += gridDim.x) {
        const int64_t a = src[s], b = dst[s], l = len[s];
        for (int64_t t = threadIdx.x; t < l; t += blockDim.x) to[b + t] = from[a + t];
    }
}

}  // namespace

extern "C" {

// Host-only routing plan (no GPU needed; tested on CPU with gloo, tests/test_exchange_gloo.py).
//   counts[2*world]          (n_seqs_r, n_tokens_r) per rank
//   offs_all[world*(max_seqs+1)]  rank r's seq offsets (relative to its token segment) at r*(max_seqs+1)
//   prompts_all[world*max_seqs]
// Sequences of rank r are at token positions r*max_tokens + offs in the gathered buffer.
// Output, in (rank, seq) order, the kept sequences (prompt % world == rank):
//   plan_src[i], plan_dst[i], plan_len[i], plan_prompt[i]; *nkeep; *ntok.
// Arrays must hold at least sum_r n_seqs_r entries.  Returns 0, or 1 on bad input.
int bs_route_plan(int32_t world, int32_t rank, const int64_t* counts, const int64_t* offs_all,
                  const int32_t* prompts_all, int64_t max_seqs, int64_t max_tokens,
                  int64_t* plan_src, int64_t* plan_dst, int64_t* plan_len, int32_t* plan_prompt,
                  int32_t* nkeep, int64_t* ntok) {
    if (world < 1 || rank < 0 || rank >= world || !counts || !nkeep || !ntok) return 1;
    int32_t k = 0;
    int64_t dst = 0;
    for (int r = 0; r < world; ++r) {
        const int64_t ns = counts[2 * r];
        if (ns < 0 || ns > max_seqs) return 1;
        const int64_t* off = offs_all + (int64_t)r * (max_seqs + 1);
        for (int64_t s = 0; s < ns; ++s) {
            const int32_t P = prompts_all[(int64_t)r * max_seqs + s];
            const int32_t owner = (int32_t)(((int64_t)P % world + world) % world);
            if (owner != rank) continue;
            const int64_t len = off[s + 1] - off[s];
            if (len < 0 || off[s + 1] > max_tokens) return 1;
            plan_src[k] = (int64_t)r * max_tokens + off[s];
            plan_dst[k] = dst;
            plan_len[k] = len;
            plan_prompt[k] = P;
            dst += len;
            ++k;
        }
    }
    *nkeep = k;
    *ntok = dst;
    return 0;
}

bs_status bs_nccl_unique_id(void* id128) {
    NcclApi& a = nccl();
    if (!a.ok) return BS_ERR_NCCL;
    ncclUniqueId id;
    if (a.GetUniqueId(&id) != ncclSuccess) return BS_ERR_NCCL;
    memcpy(id128, &id, sizeof id);
    return BS_OK;
}

bs_status bs_nccl_comm_init(void** comm_out, const void* id128, int32_t world, int32_t rank) {
    NcclApi& a = nccl();
    if (!a.ok || !comm_out) return BS_ERR_NCCL;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    ncclComm_t comm;
    if (a.CommInitRank(&comm, world, id, rank) != ncclSuccess) return BS_ERR_NCCL;
    *comm_out = comm;
    return BS_OK;
}

bs_status bs_nccl_comm_destroy(void* comm) {
    NcclApi& a = nccl();
    if (!a.ok) return BS_ERR_NCCL;
    return a.CommDestroy((ncclComm_t)comm) == ncclSuccess ? BS_OK : BS_ERR_NCCL;
}

bs_status bs_draft_exchange(bs_ctx* c, void* comm_v, int32_t rank, int32_t world, uint64_t rl_step,
                            void* stream) {
    if (!c || !comm_v || world < 1 || rank < 0 || rank >= world) return BS_ERR_INVALID;
    NcclApi& a = nccl();
    if (!a.ok) {
        c->err = "NCCL library not found";
        return BS_ERR_NCCL;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ncclComm_t comm = (ncclComm_t)comm_v;
    bs::DeviceScope dev_scope_(c->cfg.device);
    if (dev_scope_.err != cudaSuccess) return BS_ERR_CUDA;
    Pool& P = c->staging;
    if (!P.valid || P.step != rl_step) {
        P.valid = true;
        P.step = rl_step;
        P.n_seqs = 0;
        P.n_tokens = 0;
        if (bs::set_cur_step(c, rl_step, st) != cudaSuccess) return BS_ERR_CUDA;
    }
    // 1. counts
    AsyncBuf<int64_t> cnt;  // stream-ordered scratch (no synchronising cudaMalloc / cudaFree)
    if (cnt.alloc(2 * (size_t)(world + 1), st) != cudaSuccess) return BS_ERR_OOM;
    int64_t mine[2] = {P.n_seqs, P.n_tokens};
    cudaMemcpyAsync(cnt.p + 2 * world, mine, sizeof mine, cudaMemcpyHostToDevice, st);
    if (a.AllGather(cnt.p + 2 * world, cnt.p, 2, ncclInt64, comm, st) != ncclSuccess) {
        c->err = "ncclAllGather(counts) failed";
        return BS_ERR_NCCL;
    }
    std::vector<int64_t> counts(2 * (size_t)world);
    cudaMemcpyAsync(counts.data(), cnt.p, sizeof(int64_t) * 2 * world, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return BS_ERR_CUDA;
    int64_t max_seqs = 0, max_tok = 0, tot_seqs = 0;
    for (int r = 0; r < world; ++r) {
        max_seqs = std::max(max_seqs, counts[2 * r]);
        max_tok = std::max(max_tok, counts[2 * r + 1]);
        tot_seqs += counts[2 * r];
    }
    // 2. padded payload all-gather (offsets, prompt ids, tokens) in one NCCL group
    AsyncBuf<int64_t> soff, roff;
    AsyncBuf<int32_t> sprm, rprm, stok, rtok;
    if (soff.alloc(max_seqs + 1, st) || roff.alloc((size_t)world * (max_seqs + 1), st) ||
        sprm.alloc(std::max<int64_t>(max_seqs, 1), st) ||
        rprm.alloc((size_t)world * std::max<int64_t>(max_seqs, 1), st) ||
        stok.alloc(std::max<int64_t>(max_tok, 1), st) ||
        rtok.alloc((size_t)world * std::max<int64_t>(max_tok, 1), st))
        return BS_ERR_OOM;
    cudaMemsetAsync(soff.p, 0, sizeof(int64_t) * (max_seqs + 1), st);
    if (P.n_seqs) {
        cudaMemcpyAsync(soff.p, P.seq_off.p, sizeof(int64_t) * (P.n_seqs + 1), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(sprm.p, P.seq_prompt.p, sizeof(int32_t) * P.n_seqs, cudaMemcpyDeviceToDevice, st);
    }
    if (P.n_tokens)
        cudaMemcpyAsync(stok.p, P.tokens.p, sizeof(int32_t) * P.n_tokens, cudaMemcpyDeviceToDevice, st);
    a.GroupStart();
    ncclResult_t r1 = a.AllGather(soff.p, roff.p, (size_t)max_seqs + 1, ncclInt64, comm, st);
    ncclResult_t r2 = max_seqs ? a.AllGather(sprm.p, rprm.p, (size_t)max_seqs, ncclInt32, comm, st) : ncclSuccess;
    ncclResult_t r3 = max_tok ? a.AllGather(stok.p, rtok.p, (size_t)max_tok, ncclInt32, comm, st) : ncclSuccess;
    ncclResult_t r4 = a.GroupEnd();
    if (r1 != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess || r4 != ncclSuccess) {
        c->err = "ncclAllGather(payload) failed";
        return BS_ERR_NCCL;
    }
    // 3. route (host plan over the small metadata) and gather the kept payload on device
    std::vector<int64_t> offs((size_t)world * (max_seqs + 1));
    std::vector<int32_t> prm((size_t)world * std::max<int64_t>(max_seqs, 1));
    cudaMemcpyAsync(offs.data(), roff.p, sizeof(int64_t) * offs.size(), cudaMemcpyDeviceToHost, st);
    if (max_seqs)
        cudaMemcpyAsync(prm.data(), rprm.p, sizeof(int32_t) * prm.size(), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return BS_ERR_CUDA;
    // staging offsets are absolute from 0 in each rank's segment (put appends from 0)
    std::vector<int64_t> src(tot_seqs + 1), dst(tot_seqs + 1), len(tot_seqs + 1);
    std::vector<int32_t> pp(tot_seqs + 1);
    int32_t nkeep = 0;
    int64_t ntok = 0;
    if (bs_route_plan(world, rank, counts.data(), offs.data(), prm.data(), max_seqs, max_tok, src.data(),
                      dst.data(), len.data(), pp.data(), &nkeep, &ntok))
        return BS_ERR_INVALID;
    if (ntok > c->cfg.pool_capacity_tokens || nkeep > c->cfg.pool_capacity_seqs) {
        c->err = "exchange: routed pool exceeds capacity";
        return BS_ERR_CAPACITY;
    }
    AsyncBuf<int64_t> dplan;
    if (dplan.alloc(3 * (size_t)std::max(nkeep, 1), st)) return BS_ERR_OOM;
    cudaMemcpyAsync(dplan.p, src.data(), sizeof(int64_t) * nkeep, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dplan.p + nkeep, dst.data(), sizeof(int64_t) * nkeep, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dplan.p + 2 * nkeep, len.data(), sizeof(int64_t) * nkeep, cudaMemcpyHostToDevice, st);
    if (nkeep)
        gather_seqs_kernel<<<std::min(nkeep, 4096), 256, 0, st>>>(nkeep, dplan.p, dplan.p + nkeep,
                                                                 dplan.p + 2 * nkeep, rtok.p, P.tokens.p);
    std::vector<int64_t> new_off(nkeep + 1);
    for (int i = 0; i < nkeep; ++i) new_off[i] = dst[i];
    new_off[nkeep] = ntok;
    cudaMemcpyAsync(P.seq_off.p, new_off.data(), sizeof(int64_t) * (nkeep + 1), cudaMemcpyHostToDevice, st);
    if (nkeep)
        cudaMemcpyAsync(P.seq_prompt.p, pp.data(), sizeof(int32_t) * nkeep, cudaMemcpyHostToDevice, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return BS_ERR_CUDA;
    P.n_seqs = nkeep;
    P.n_tokens = ntok;
    return BS_OK;
}

}  // extern "C"
