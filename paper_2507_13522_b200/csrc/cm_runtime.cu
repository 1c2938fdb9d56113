// cm_runtime.cu -- host runtime and C ABI of libcm.so (see include/cm.h for the contract).
//
// One context per rank.  Responsibilities: bucket planning, peer
// mapping over CUDA IPC (NVLink), the POSIX-shm shadow segment (tap ring + shadow state,
// the analog of the paper's shadow cluster), stream/event
// orchestration for flow control, and kernel launches.  Every
// numerical step runs in the sm_100a kernels of cm_kernels.cuh; this file only moves
// pointers, computes the per-step fp32 scalars (reading R5/R6) and sequences work.
#include "cm.h"
#include "cm_kernels.cuh"
#include "cm_segment.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <poll.h>
#include <sys/mman.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

using namespace cm;
static_assert(kSegMaxRanks == kMaxRanks, "rank bound");

// segment layout, SegHeader, SlotMeta: cm_segment.h
namespace {

constexpr int kStages = 4;                       // shadow staging buffers
constexpr int64_t kOsSlotBytes = 1ll << 20;      // one-shot inbox slot (largest one-shot bucket)
constexpr int64_t kDrainCoalesce = 64ll << 20;   // tap drains of adjacent shards merge up to this
constexpr int64_t kStageElems = 8ll << 20;       // elements per shadow staging chunk

uint64_t process_token() {
    static uint64_t tok = [] {
        std::random_device rd;
        return ((uint64_t)rd() << 32) ^ rd() ^ ((uint64_t)getpid() << 16);
    }();
    return tok;
}

// Exchange blob: what a rank tells its peers.
struct Blob {
    uint64_t magic;
    uint64_t token;         // process identity: equal tokens = same process
    int32_t world_size, rank, device, dtype;
    uint64_t layout_hash;
    int64_t padded_numel;
    // 0 grad, 1 p, 2 m, 3 v, 4 signal pad, 5 one-shot inbox
    cudaIpcMemHandle_t handle[6];
    uint64_t base[6];       // allocation base address in the owner (dedupe key)
    uint64_t offset[6];     // pointer - base
    uint64_t raw[6];        // raw pointer (usable in-process)
};

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

// One step's optimizer and scalars: what the trainer used, what the shadow and the
// restore roll-forward replay (the ring-slot record holds the same ten floats + kind).
struct StepRec {
    int kind = kOptAdamW;
    AdamScalars a{};
    SgdScalars q{};
    void to_floats(float* f) const {
        memset(f, 0, 10 * sizeof(float));
        if (kind == kOptAdamW) memcpy(f, &a, sizeof a);
        else { f[0] = q.mu; f[1] = q.inv_n; f[2] = q.lr; f[3] = q.wd; f[4] = q.wd_on ? 1.0f : 0.0f; }
    }
    static StepRec from_floats(int kind, const float* f) {
        StepRec r;
        r.kind = kind;
        if (kind == kOptAdamW) memcpy(&r.a, f, sizeof r.a);
        else { r.q.mu = f[0]; r.q.inv_n = f[1]; r.q.lr = f[2]; r.q.wd = f[3]; r.q.wd_on = f[4] != 0.0f; }
        return r;
    }
};
static_assert(sizeof(AdamScalars) == 10 * sizeof(float), "record");

}  // namespace

struct cm_ctx {
    cm_config cfg{};
    std::string shm_name;
    std::string err;
    int n = 1, rank = 0, dev = 0, D = 2, dtype = 0, es = 4;
    bool no_tap = false, attach = false, ce_tap = false, no_shadow = false, staged_tap = false;
    bool zero1 = false;                   // CM_FLAG_ZERO1: sharded optimizer state
    int zero1_blocks = 296;
    int zero1_tma_blocks = 592;
    void* stage_buf[2] = {};              // default tap: HBM staging of the reduced shard
    cudaEvent_t ev_stage_free[2] = {};    // staging half drained to the host ring
    cudaEvent_t ev_ar_done[2] = {};       // all all-reduce kernels of the half's iteration done
    cudaEvent_t ev_stage_consumed[2] = {};// the shadow step reading the half from HBM is done
    bool stage_consumer[2] = {false, false};
    int64_t stage_iter[2] = {-1, -1};     // iteration whose reduced shard the half holds
    int shadow_place = CM_SHADOW_HOST;
    int sms = 148;
    bool cuda_dead = false;

    // plan
    bool registered = false, connected = false;
    std::vector<int64_t> numel;
    int64_t cap_bytes = 0;
    std::vector<BucketDev> buckets;
    int64_t P_pad = 0, shard_numel = 0;
    uint64_t layout_hash = 0;
    BucketDev* d_buckets = nullptr;

    // user buffers (this rank) and peers
    void* grad = nullptr;
    float *p = nullptr, *m = nullptr, *v = nullptr;
    uint32_t* pad = nullptr;
    char* inbox = nullptr;                // one-shot inbox: 2 halves x n slots x kOsSlotBytes
    char* peer_inbox[kMaxRanks] = {};
    // NVLS (CM_FLAG_NVLS): the inbox is physical memory bound to a multicast object; pushes
    // go through the multicast mapping mc_va, reads through the unicast mapping uc_va
    bool nvls = false;
    CUmemGenericAllocationHandle mc_handle = 0, mc_phys = 0;
    CUdeviceptr mc_va = 0, uc_va = 0;
    size_t mc_size = 0;
    int64_t oneshot_max = 0;              // buckets <= this many bytes use the one-shot kernel
    bool ablate_no_drain = false;         // ablation only: staged taps never reach the host ring
    bool lazy_exit = true;                // all-reduce kernels without exit barrier; the training
                                          // step's entry barrier fences the iteration instead
    int64_t drain_flush = 8ll << 20;      // a pending drain run is issued once it holds this much
    int drain_ctas = -1;                  // D2H of tap drains / persists: 0 copy engine, k>0 k-CTA SM
                                          // drain, -1 auto (SM drain when the link demand is low)
    int numa_req = -2;                    // host segment placement: -2 the GPU's NUMA node (auto),
                                          // -1 kernel default (first touch), k >= 0 node k
    int numa_used = -1;                   // node the segment was bound to (-1: none)
    double iter_period_s = 0.0;           // EMA of the GPU's period between training steps
    static constexpr int kStepEv = 8;     // events recorded after each step's optimizer kernel
    cudaEvent_t ev_gstep[kStepEv] = {};
    int64_t ev_gstep_step[kStepEv] = {-1, -1, -1, -1, -1, -1, -1, -1};
    int64_t gper_last = 0;                // newest step whose period went into the estimate
    char* peer_grad[kMaxRanks] = {};
    float* peer_p[kMaxRanks] = {};
    float* peer_m[kMaxRanks] = {};
    float* peer_v[kMaxRanks] = {};
    Pads pads{};
    std::vector<std::pair<uint64_t, void*>> opened;  // (peer base key, mapped ptr)
    bool in_process = false, barriers = true;
    uint32_t epoch = 0;
    unsigned long long* d_done_ctr = nullptr;            // [n_buckets]: blocks finished (direct tap)
    std::vector<unsigned long long> done_total;          // per bucket: cumulative launch blocks
    unsigned long long* d_bad = nullptr;
    // non-finite report pair (step, index): host view + device alias.  Points into the segment
    // header once connected with a tap (it then survives the process), else into `ctl`.
    int64_t* ctl = nullptr;               // pinned, mapped fallback pair
    volatile int64_t* nf_host = nullptr;
    volatile int64_t* nf_dev = nullptr;   // device alias of nf_host (host-mapped)
    int64_t* d_nf = nullptr;              // device word: the flagged step (read by shadow kernels)
    NfRef nfref() const { return NfRef{nf_dev, (volatile int64_t*)d_nf}; }
    // cm_verify_ex scratch (chunked host roll-forward): p, m, v chunks
    float* vf_scratch = nullptr;

    // launch geometry
    int ar_blocks_max = 296, adam_blocks = 1184, shadow_blocks = 296, misc_blocks = 1184;
    int ar_blocks_tap_only = 32;   // n == 1: the kernel is only the PCIe tap; leave SMs free
    int adamw_impl = 2;            // 0 vectorised, 1 TMA bulk-copy staged, 2 warp-tiled (measured best)
    int ar_impl = -1;              // -1 auto (bulk-copy pipeline from ar_tma_min bytes, else the
                                   // unrolled kernel), 0 unrolled two-shot, 1 software-pipelined
                                   // (one block per SM), 2 bulk-copy (TMA) pipeline always
    int64_t ar_tma_min = 12ll << 20;   // auto: buckets of at least this many bytes take the bulk
                                       // copies (measured: faster from 16 MiB, slower at 4-8 MiB)
    int ar_tma_tile_req = 0;           // bulk-copy tile bytes per rank per stage (0: by n)
    int ar_tma_stages = 2;             // bulk-copy pipeline depth (2 or 3)
    int zero1_impl = 1;            // ZeRO-1 AdamW + AG: 1 two groups per thread in flight, 0 one,
                                   // 2 tiles pushed by bulk copies (cp.async.bulk)
    int ar_pipe_blocks = 148;
    int ar_blocks_user = 0;        // ar_blocks set explicitly: no size-dependent grid
    int64_t ar_grid_switch = 48ll << 20;   // buckets up to this many bytes: one block per SM
    bool pdl = false;              // programmatic dependent launch of the all-reduce kernels
    int pdl_mode = 0;              // experiments (see ArParams::pdl_mode)
    bool pdl_force = false;        // test only: PDL even with exit barriers (deadlock regression)
    bool force_no_barriers = false;   // profiling only: in-process ranks on several GPUs without
                                      // the cross-GPU barriers (ncu serialises kernels; values
                                      // are then meaningless, the NVLink traffic is real)
    bool persist_on_tap = false;   // snapshot persists on the tap-drain stream (one D2H queue)
    bool n1_ce_stage = false;      // n == 1: a copy engine copies each bucket into staging
    bool shadow_after_train = true;   // the shadow step waits for the training step's optimizer
                                      // (measured: -0.2 ms per GPT-2 step at n=1, profiles/r02/
                                      // r02u_model_n1_shadow_after_train_ab.jsonl)
    cudaStream_t last_s = nullptr; // stream of this context's latest launch on a caller stream,
    int last_kind = 0;             // and its kind (1: an all-reduce kernel, 0: anything else)
    int64_t last_iter = -1;        // iteration of that all-reduce kernel
    int tma_blocks = 148;
    int wt_blocks = 296;
    int wt1_blocks = 592;

    // shadow segment
    int shm_fd = -1;
    char* seg = nullptr;
    size_t seg_size = 0;
    bool seg_registered = false;
    char* seg_dev = nullptr;      // device alias of the mapped segment
    SegHeader* hdr = nullptr;
    // The shadow's working state lives in HBM as two ping-pong halves (half s&1 holds step
    // s) outside the training buffers; with HOST placement every step is also persisted to
    // the matching host half in the shm segment (write-through), so the host copy alone
    // survives the process and the GPU.
    float* state_dev_alloc = nullptr;
    float* sd[2][3] = {};               // HBM halves {p, m, v}
    float* sh[2][3] = {};               // host halves (HOST placement), nullptr otherwise

    // iteration bookkeeping
    int64_t cur_iter = 0;
    std::vector<char> issued;
    int issued_count = 0;
    // per-bucket optimizer steps (cm_apply_bucket) of the current iteration
    std::vector<char> applied;
    int applied_count = 0;
    StepRec bucket_rec;                 // the step's scalars, fixed by its first bucket
    int64_t grads_step = -1;            // the training step whose reduced gradients the grad
                                        // buffer / staging hold (-1 after a restore)
    int64_t train_step = 0;
    int64_t shadow_enq = 0;
    int K = 1;                       // persist the host snapshot every K shadow steps
    int64_t released_upto = 0;       // ring slots of iterations < released_upto are free
    int64_t hh_step[2] = {0, -1};    // host snapshot halves' steps (enqueue-time mirror)
    int opt_kind = -1;               // optimizer fixed by the first step (-1: none yet)
    std::vector<StepRec> slot_sc;
    std::vector<int64_t> slot_sc_step;
    std::vector<cudaEvent_t> ev_tap_done, ev_slot_free;

    // scalar cache (reading R6: beta^s by repeated multiplication from 1.0)
    double pw_b1 = 1.0, pw_b2 = 1.0, pw_beta1 = -1, pw_beta2 = -1;
    int64_t pw_s = 0;

    int64_t launches = 0;

    // pending (not yet issued) copy-engine drain of adjacent tapped shards [dr_b0, dr_b1]
    int dr_b0 = -1, dr_b1 = -1;
    int64_t dr_iter = -1;
    const char* dr_src = nullptr;
    char* dr_dst = nullptr;
    size_t dr_bytes = 0;

    // copy-engine staging of the shadow step (shadow_step_enqueue)
    bool stg_ready = false;
    cudaStream_t cs_h2d = nullptr, cs_d2h = nullptr, cs_k = nullptr;
    cudaStream_t cs_tap = nullptr;   // CM_FLAG_TAP_COPYENGINE
    cudaEvent_t ev_ar = nullptr;
    int64_t stg_elems = 0;
    void* stg_g[4] = {};
    cudaEvent_t ev_stg_free[4] = {}, ev_stg_ready[4] = {}, ev_fork = nullptr, ev_join = nullptr;

    // optional per-kernel timing (cm_timing): event pairs on the launching stream
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> timed;  // (class, (start, end))
    int64_t timed_bytes[7] = {};     // device->host bytes of classes 5 / 6 in the window
    int64_t last_bytes[7] = {};      // ... of the last closed window (cm_timing_bytes)
};

// ====================================================================== helpers
static int ar_tma_tile(const cm_ctx* c) {
    int t = c->ar_tma_tile_req;
    if (t <= 0) t = ArTma<2>::kTile;
    const int cap = (kArTmaMaxSmem / (c->ar_tma_stages * c->n)) / 128 * 128;
    return std::max(128, std::min(t, cap));
}

static cm_status fail(cm_ctx* c, cm_status s, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    if (c && s == CM_ERR_CUDA) c->cuda_dead = true;
    return s;
}

#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(c, CM_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                              \
    } while (0)

#define CHECK_LAUNCH() CU(cudaGetLastError())

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

// The non-finite report (reading R16) as a status: CM_ERR_INVARIANT once a kernel reported
// an inf/NaN, until cm_restore rolls back to the last finite step.  Read from host-mapped
// memory, no synchronisation.  Collective calls never refuse because of it: ranks observe
// the report at different times, and a rank that refused a collective its peers issued would
// leave their kernels waiting at a barrier.  The device side makes the report safe instead
// (the shadow never applies or publishes the flagged step; restore never rolls forward to
// it); callers poll cm_check (and agree across ranks, as with a loss-scaler's found-inf) or
// see it from cm_verify_ex.
static cm_status check_nf(cm_ctx* c) {
    if (!c->nf_host) return CM_OK;
    const int64_t st = c->nf_host[0];
    if (st < 0) return CM_OK;
    return fail(c, CM_ERR_INVARIANT,
                "non-finite value (inf/NaN) in step %lld at flat index %lld; the shadow stopped at the last "
                "finite step: call cm_restore", (long long)st, (long long)c->nf_host[1]);
}

// ---------------------------------------------------------------- bucket planner
// PAPER.md:258-264 (sec 4.2.2) with readings R10-R13 (see cm.h cm_plan_buckets).
struct PlanOut {
    std::vector<BucketDev> buckets;
    std::vector<int64_t> tensor_off;
    int64_t total = 0;
};

static bool plan(const int64_t* numel, int nt, int64_t cap, int es, int n, PlanOut& out) {
    if (nt <= 0 || cap <= 0 || n <= 0 || (es != 2 && es != 4)) return false;
    for (int i = 0; i < nt; ++i)
        if (numel[i] <= 0) return false;
    const int64_t quantum = (16 / es) * (int64_t)n;
    std::vector<std::vector<int>> groups;
    int64_t open_bytes = -1;  // -1: no open bucket
    for (int i = nt - 1; i >= 0; --i) {
        const int64_t bytes = numel[i] * es;
        if (bytes > cap) {
            groups.push_back({i});
            open_bytes = -1;
        } else if (open_bytes >= 0 && open_bytes + bytes <= cap) {
            groups.back().push_back(i);
            open_bytes += bytes;
        } else {
            groups.push_back({i});
            open_bytes = bytes;
        }
    }
    out.tensor_off.assign(nt, 0);
    out.buckets.clear();
    int64_t flat = 0;
    for (auto& g : groups) {
        BucketDev b{};
        b.off = flat;
        int64_t used = 0;
        for (int i : g) {
            out.tensor_off[i] = flat + used;
            used += numel[i];
        }
        b.used = used;
        b.padded = (used + quantum - 1) / quantum * quantum;
        b.shard_off = flat / n;
        out.buckets.push_back(b);
        flat += b.padded;
    }
    out.total = flat;
    return true;
}


// ---------------------------------------------------------------- AdamW scalars
// Reading R5: fp64 arithmetic, one rounding to fp32 per scalar; R6: beta^s by s
// repeated fp64 multiplications from 1.0 (cached incrementally: the same sequence).
static AdamScalars make_scalars(cm_ctx* c, int64_t s, const cm_adamw& hp) {
    if (hp.beta1 != c->pw_beta1 || hp.beta2 != c->pw_beta2 || s < c->pw_s) {
        c->pw_b1 = 1.0; c->pw_b2 = 1.0; c->pw_s = 0;
        c->pw_beta1 = hp.beta1; c->pw_beta2 = hp.beta2;
    }
    while (c->pw_s < s) {
        c->pw_b1 = c->pw_b1 * hp.beta1;
        c->pw_b2 = c->pw_b2 * hp.beta2;
        c->pw_s++;
    }
    AdamScalars a;
    a.c1 = (float)(1.0 - hp.beta1);
    a.c2 = (float)(1.0 - hp.beta2);
    a.B1 = (float)hp.beta1;
    a.B2 = (float)hp.beta2;
    a.bc1 = (float)(1.0 - c->pw_b1);
    a.bc2 = (float)(1.0 - c->pw_b2);
    a.inv_n = (float)(1.0 / (double)c->n);
    a.lr = (float)hp.lr;
    a.eps = (float)hp.eps;
    a.wd = (float)hp.weight_decay;
    return a;
}

// SGD-momentum scalars (reading R27): fp64 -> fp32 once; wd_on decided on the host
static SgdScalars make_sgd_scalars(cm_ctx* c, const cm_sgd& hp) {
    SgdScalars q;
    q.mu = (float)hp.momentum;
    q.inv_n = (float)(1.0 / (double)c->n);
    q.lr = (float)hp.lr;
    q.wd = (float)hp.weight_decay;
    q.wd_on = hp.weight_decay != 0.0 ? 1 : 0;
    return q;
}

// ---------------------------------------------------------------- launch helpers
template <typename G, int N>
static int ar_occ_n() {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rs_tap_ag_kernel<G, N>, kArThreads, 0);
    return occ > 0 ? occ : 1;
}
// co-resident blocks per SM of the n-rank instance (blocks pair across GPUs by index, so
// the grid never exceeds what is resident at once)
template <typename G>
static int ar_occupancy(int n) {
    switch (n) {
        case 1: return ar_occ_n<G, 1>();
        case 2: return ar_occ_n<G, 2>();
        case 3: return ar_occ_n<G, 3>();
        case 4: return ar_occ_n<G, 4>();
        case 5: return ar_occ_n<G, 5>();
        case 6: return ar_occ_n<G, 6>();
        case 7: return ar_occ_n<G, 7>();
        default: return ar_occ_n<G, 8>();
    }
}

template <typename G>
static void launch_ar_pipe_t(int n, dim3 grid, cudaStream_t s, const ArParams& P) {
    switch (n) {
        case 1: rs_tap_ag_pipe_kernel<G, 1><<<grid, kArThreads, 0, s>>>(P); break;
        case 2: rs_tap_ag_pipe_kernel<G, 2><<<grid, kArThreads, 0, s>>>(P); break;
        case 3: rs_tap_ag_pipe_kernel<G, 3><<<grid, kArThreads, 0, s>>>(P); break;
        case 4: rs_tap_ag_pipe_kernel<G, 4><<<grid, kArThreads, 0, s>>>(P); break;
        case 5: rs_tap_ag_pipe_kernel<G, 5><<<grid, kArThreads, 0, s>>>(P); break;
        case 6: rs_tap_ag_pipe_kernel<G, 6><<<grid, kArThreads, 0, s>>>(P); break;
        case 7: rs_tap_ag_pipe_kernel<G, 7><<<grid, kArThreads, 0, s>>>(P); break;
        default: rs_tap_ag_pipe_kernel<G, 8><<<grid, kArThreads, 0, s>>>(P); break;
    }
}

// launch with programmatic stream serialization (PDL) when pdl is set (see cm_kernels.cuh)
static cudaError_t launch_pdl(void (*k)(ArParams), dim3 grid, cudaStream_t s, bool pdl, const ArParams& P,
                              int threads = kArThreads, size_t smem = 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? at : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, P);
}

template <typename G, int N>
static void set_ar_tma_smem() {
    cudaFuncSetAttribute(rs_tap_ag_tma_kernel<G, N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kArTmaMaxSmem);
    cudaFuncSetAttribute(rs_tap_ag_tma_kernel<G, N, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kArTmaMaxSmem);
}
template <typename G>
static void set_ar_tma_smem_all() {
    set_ar_tma_smem<G, 2>(); set_ar_tma_smem<G, 3>(); set_ar_tma_smem<G, 4>(); set_ar_tma_smem<G, 5>();
    set_ar_tma_smem<G, 6>(); set_ar_tma_smem<G, 7>(); set_ar_tma_smem<G, 8>();
}
template <typename G, int N>
static void launch_ar_tma_n(dim3 grid, cudaStream_t s, const ArParams& P, bool pdl, int stages) {
    const size_t smem = (size_t)stages * N * P.tma_tile;
    if (stages == 3) launch_pdl(rs_tap_ag_tma_kernel<G, N, 3>, grid, s, pdl, P, kArTmaThreads, smem);
    else launch_pdl(rs_tap_ag_tma_kernel<G, N, 2>, grid, s, pdl, P, kArTmaThreads, smem);
}
template <typename G>
static void launch_ar_tma_t(int n, dim3 grid, cudaStream_t s, const ArParams& P, bool pdl, int stages) {
    switch (n) {
        case 2: launch_ar_tma_n<G, 2>(grid, s, P, pdl, stages); break;
        case 3: launch_ar_tma_n<G, 3>(grid, s, P, pdl, stages); break;
        case 4: launch_ar_tma_n<G, 4>(grid, s, P, pdl, stages); break;
        case 5: launch_ar_tma_n<G, 5>(grid, s, P, pdl, stages); break;
        case 6: launch_ar_tma_n<G, 6>(grid, s, P, pdl, stages); break;
        case 7: launch_ar_tma_n<G, 7>(grid, s, P, pdl, stages); break;
        default: launch_ar_tma_n<G, 8>(grid, s, P, pdl, stages); break;
    }
}
// bytes per rank per stage: the configured tile, capped so stages x n x tile fits the smem cap
static int ar_tma_tile(const cm_ctx* c);

template <typename G>
static void launch_ar_t(int n, dim3 grid, cudaStream_t s, const ArParams& P, bool pdl) {
    void (*k)(ArParams) = nullptr;
    switch (n) {
        case 1: k = rs_tap_ag_kernel<G, 1>; break;
        case 2: k = rs_tap_ag_kernel<G, 2>; break;
        case 3: k = rs_tap_ag_kernel<G, 3>; break;
        case 4: k = rs_tap_ag_kernel<G, 4>; break;
        case 5: k = rs_tap_ag_kernel<G, 5>; break;
        case 6: k = rs_tap_ag_kernel<G, 6>; break;
        case 7: k = rs_tap_ag_kernel<G, 7>; break;
        default: k = rs_tap_ag_kernel<G, 8>; break;
    }
    launch_pdl(k, grid, s, pdl, P);
}

template <typename G>
static void launch_os_t(int n, int grid, cudaStream_t s, const OsParams& P) {
    switch (n) {
        case 2: os_tap_kernel<G, 2><<<grid, kOsThreads, 0, s>>>(P); break;
        case 3: os_tap_kernel<G, 3><<<grid, kOsThreads, 0, s>>>(P); break;
        case 4: os_tap_kernel<G, 4><<<grid, kOsThreads, 0, s>>>(P); break;
        case 5: os_tap_kernel<G, 5><<<grid, kOsThreads, 0, s>>>(P); break;
        case 6: os_tap_kernel<G, 6><<<grid, kOsThreads, 0, s>>>(P); break;
        case 7: os_tap_kernel<G, 7><<<grid, kOsThreads, 0, s>>>(P); break;
        default: os_tap_kernel<G, 8><<<grid, kOsThreads, 0, s>>>(P); break;
    }
}

static cm_status launch_adamw(cm_ctx* c, const AdamParams& P, int blocks, cudaStream_t s) {
    if (P.rec_kind == kOptSgd) {
        // SGD-momentum: the warp-tiled data path only
        const int64_t tiles = P.n / kWarpTile;
        const int64_t want = std::max<int64_t>(1, (tiles + kAdamThreads / 32 - 1) / (kAdamThreads / 32));
        const int grid = (int)std::min<int64_t>(want, std::min(blocks, c->wt_blocks));
        if (c->dtype == CM_F32) sgd_wt_kernel<F32Tag><<<grid, kAdamThreads, 0, s>>>(P);
        else sgd_wt_kernel<BF16Tag><<<grid, kAdamThreads, 0, s>>>(P);
    } else if (c->adamw_impl == 1 && !P.fence_n) {   // (the iteration fence lives in the warp-tiled body)
        const int64_t tiles = (P.n + kTmaTile - 1) / kTmaTile;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, c->tma_blocks));
        if (c->dtype == CM_F32)
            adamw_tma_kernel<F32Tag><<<grid, kTmaThreads, kTmaStages * TmaTile<F32Tag>::kStageBytes, s>>>(P);
        else
            adamw_tma_kernel<BF16Tag><<<grid, kTmaThreads, kTmaStages * TmaTile<BF16Tag>::kStageBytes, s>>>(P);
    } else if (c->adamw_impl == 3) {
        const int64_t tiles = P.n / kWarpTile;
        const int64_t want = std::max<int64_t>(1, (tiles + kAdamThreads / 32 - 1) / (kAdamThreads / 32));
        const int grid = (int)std::min<int64_t>(want, c->wt1_blocks);
        if (c->dtype == CM_F32) adamw_wt1_kernel<F32Tag><<<grid, kAdamThreads, 0, s>>>(P);
        else adamw_wt1_kernel<BF16Tag><<<grid, kAdamThreads, 0, s>>>(P);
    } else if (c->adamw_impl == 2 || P.fence_n) {
        const int64_t tiles = P.n / kWarpTile;
        const int64_t want = std::max<int64_t>(1, (tiles + kAdamThreads / 32 - 1) / (kAdamThreads / 32));
        const int grid = (int)std::min<int64_t>(want, std::min(blocks, c->wt_blocks));
        if (c->dtype == CM_F32) adamw_wt_kernel<F32Tag><<<grid, kAdamThreads, 0, s>>>(P);
        else adamw_wt_kernel<BF16Tag><<<grid, kAdamThreads, 0, s>>>(P);
    } else {
        int64_t items = P.n / 8;
        int64_t want = (items + kAdamThreads - 1) / kAdamThreads;
        int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, blocks));
        if (c->dtype == CM_F32) adamw_kernel<F32Tag><<<grid, kAdamThreads, 0, s>>>(P);
        else adamw_kernel<BF16Tag><<<grid, kAdamThreads, 0, s>>>(P);
    }
    c->launches++;
    CHECK_LAUNCH();
    return CM_OK;
}

template <typename G, int OPT>
static void launch_zero1_tma_t(int n, int grid, cudaStream_t s, const Zero1Params& Z) {
    switch (n) {
        case 1: adamw_zero1_tma_kernel<G, 1, OPT><<<grid, kZ1TmaThreads, 0, s>>>(Z); break;
        case 2: adamw_zero1_tma_kernel<G, 2, OPT><<<grid, kZ1TmaThreads, 0, s>>>(Z); break;
        case 3: adamw_zero1_tma_kernel<G, 3, OPT><<<grid, kZ1TmaThreads, 0, s>>>(Z); break;
        case 4: adamw_zero1_tma_kernel<G, 4, OPT><<<grid, kZ1TmaThreads, 0, s>>>(Z); break;
        case 5: adamw_zero1_tma_kernel<G, 5, OPT><<<grid, kZ1TmaThreads, 0, s>>>(Z); break;
        case 6: adamw_zero1_tma_kernel<G, 6, OPT><<<grid, kZ1TmaThreads, 0, s>>>(Z); break;
        case 7: adamw_zero1_tma_kernel<G, 7, OPT><<<grid, kZ1TmaThreads, 0, s>>>(Z); break;
        default: adamw_zero1_tma_kernel<G, 8, OPT><<<grid, kZ1TmaThreads, 0, s>>>(Z); break;
    }
}
template <typename G, int OPT>
static void launch_zero1_t(int n, int grid, cudaStream_t s, const Zero1Params& Z) {
    switch (n) {
        case 1: adamw_zero1_kernel<G, 1, OPT><<<grid, 256, 0, s>>>(Z); break;
        case 2: adamw_zero1_kernel<G, 2, OPT><<<grid, 256, 0, s>>>(Z); break;
        case 3: adamw_zero1_kernel<G, 3, OPT><<<grid, 256, 0, s>>>(Z); break;
        case 4: adamw_zero1_kernel<G, 4, OPT><<<grid, 256, 0, s>>>(Z); break;
        case 5: adamw_zero1_kernel<G, 5, OPT><<<grid, 256, 0, s>>>(Z); break;
        case 6: adamw_zero1_kernel<G, 6, OPT><<<grid, 256, 0, s>>>(Z); break;
        case 7: adamw_zero1_kernel<G, 7, OPT><<<grid, 256, 0, s>>>(Z); break;
        default: adamw_zero1_kernel<G, 8, OPT><<<grid, 256, 0, s>>>(Z); break;
    }
}
static void launch_zero1(cm_ctx* c, const Zero1Params& Z, int grid, cudaStream_t s) {
    if (c->zero1_impl == 2) {   // tiles of kZ1TmaTile elements, pushed by bulk copies
        int64_t tiles = 0;
        for (const auto& B : c->buckets) tiles += (B.padded / c->n + kZ1TmaTile - 1) / kZ1TmaTile;
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, c->zero1_tma_blocks));
        if (Z.rec_kind == kOptSgd) {
            if (c->dtype == CM_F32) launch_zero1_tma_t<F32Tag, kOptSgd>(c->n, g, s, Z);
            else launch_zero1_tma_t<BF16Tag, kOptSgd>(c->n, g, s, Z);
        } else {
            if (c->dtype == CM_F32) launch_zero1_tma_t<F32Tag, kOptAdamW>(c->n, g, s, Z);
            else launch_zero1_tma_t<BF16Tag, kOptAdamW>(c->n, g, s, Z);
        }
        return;
    }
    if (Z.rec_kind == kOptSgd) {
        if (c->dtype == CM_F32) launch_zero1_t<F32Tag, kOptSgd>(c->n, grid, s, Z);
        else launch_zero1_t<BF16Tag, kOptSgd>(c->n, grid, s, Z);
    } else {
        if (c->dtype == CM_F32) launch_zero1_t<F32Tag, kOptAdamW>(c->n, grid, s, Z);
        else launch_zero1_t<BF16Tag, kOptAdamW>(c->n, grid, s, Z);
    }
}

// the params of one element-local step kernel for record r
static void set_step(AdamParams& P, const StepRec& r) {
    P.s = r.a;
    P.q = r.q;
    P.rec_kind = r.kind;
    r.to_floats(P.rec);
}

// skip_step >= 0: a conditional publication that does not happen once step skip_step (or an
// earlier one) was flagged non-finite; -1: unconditional (invalidations)
static cm_status publish(cm_ctx* c, volatile int64_t* host_field, int64_t value, cudaStream_t s,
                         int64_t skip_step = -1) {
    // device alias of a header field
    volatile int64_t* d = (volatile int64_t*)(c->seg_dev + ((char*)host_field - c->seg));
    publish_kernel<<<1, 1, 0, s>>>(d, value, skip_step >= 0 ? (const volatile int64_t*)c->d_nf : nullptr, skip_step);
    c->launches++;
    CHECK_LAUNCH();
    return CM_OK;
}

static SlotMeta* slot_meta(cm_ctx* c, int slot) {
    return (SlotMeta*)(c->seg + c->hdr->meta_off) + slot;
}
static volatile uint64_t* slot_flags(cm_ctx* c, int slot) {
    return (volatile uint64_t*)(c->seg + c->hdr->flags_off) + (size_t)slot * c->buckets.size();
}
static char* ring_slot_dev(cm_ctx* c, int slot) {
    return c->seg_dev + c->hdr->ring_off + (size_t)slot * c->shard_numel * c->es;
}
static char* ring_slot_host(cm_ctx* c, int slot) {
    return c->seg + c->hdr->ring_off + (size_t)slot * c->shard_numel * c->es;
}
template <typename T>
static T* to_dev(cm_ctx* c, T* host) {
    return (T*)(c->seg_dev + ((char*)host - c->seg));
}

// per-kernel timing: classes 0 all-reduce (rs_tap_ag), 1 train AdamW, 2 shadow AdamW,
// 3 input generation, 4 restore copy
static cudaEvent_t timing_event(cm_ctx* c) {
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}
constexpr int kTimingClasses = 7;   // cm_timing: 5 kernel classes + tap drains + persists
struct TimedScope {
    cm_ctx* c; int cls; cudaStream_t s; cudaEvent_t a = nullptr;
    TimedScope(cm_ctx* c_, int cls_, cudaStream_t s_) : c(c_), cls(cls_), s(s_) {
        if (c->timing && (a = timing_event(c))) cudaEventRecord(a, s);
    }
    ~TimedScope() {
        if (!a) return;
        cudaEvent_t b = timing_event(c);
        if (!b) return;
        cudaEventRecord(b, s);
        c->timed.push_back({cls, {a, b}});
    }
};

// ====================================================================== C ABI
extern "C" {

cm_status cm_join(cm_ctx* c, void* stream) {
    if (!c) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    cudaStream_t s = S(stream);
    cudaStream_t internal[4] = {c->cs_tap, c->cs_h2d, c->cs_d2h, c->cs_k};
    for (cudaStream_t q : internal) {
        if (!q) continue;
        cudaEvent_t e;
        CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CU(cudaEventRecord(e, q));
        CU(cudaStreamWaitEvent(s, e, 0));
        CU(cudaEventDestroy(e));
    }
    return CM_OK;
}

cm_status cm_set_param(cm_ctx* c, const char* key, int64_t value) {
    if (!c || !key) return CM_ERR_ARG;
    const std::string k = key;
    if (k == "adamw_impl" && value >= 0 && value <= 3) c->adamw_impl = (int)value;
    else if (k == "adam_blocks" && value >= 1 && value <= 65535) c->adam_blocks = (int)value;
    else if (k == "ar_blocks_tap_only" && value >= 1 && value <= kMaxBarrierBlocks) c->ar_blocks_tap_only = (int)value;
    else if (k == "shadow_blocks" && value >= 1 && value <= 65535) c->shadow_blocks = (int)value;
    else if (k == "tma_blocks" && value >= 1 && value <= 65535) c->tma_blocks = (int)value;
    else if (k == "ar_blocks" && value >= 1 && value <= kMaxBarrierBlocks) { c->ar_blocks_max = (int)value; c->ar_blocks_user = 1; }
    else if (k == "ar_grid_switch_bytes" && value >= 0) c->ar_grid_switch = value;
    else if (k == "pdl" && (value >= 0 && value <= 2)) { c->pdl = value != 0; c->pdl_force = value == 2; }
    else if (k == "pdl_mode" && value >= 0 && value <= 3) c->pdl_mode = (int)value;
    else if (k == "force_no_barriers" && (value == 0 || value == 1) && !c->connected) c->force_no_barriers = value != 0;
    else if (k == "persist_queue" && (value == 0 || value == 1)) c->persist_on_tap = value != 0;
    else if (k == "n1_copy_engine" && (value == 0 || value == 1)) c->n1_ce_stage = value != 0;
    else if (k == "shadow_after_train" && (value == 0 || value == 1)) c->shadow_after_train = value != 0;
    else if (k == "oneshot_max_bytes" && value >= 0 && value <= kOsSlotBytes) c->oneshot_max = value;
    else if (k == "drain_ctas" && value >= -1 && value <= 64) c->drain_ctas = (int)value;
    else if (k == "lazy_exit" && (value == 0 || value == 1)) c->lazy_exit = value;
    else if (k == "numa_node" && value >= -2 && value < 64 && !c->seg) c->numa_req = (int)value;
    else if (k == "drain_flush_bytes" && value >= 0 && value <= kDrainCoalesce) c->drain_flush = value;
    else if (k == "ar_impl" && value >= -1 && value <= 2) c->ar_impl = (int)value;
    else if (k == "ar_tma_min_bytes" && value >= 0) c->ar_tma_min = value;
    else if (k == "ar_tma_tile" && value >= 0 && value <= 65536 && value % 128 == 0) c->ar_tma_tile_req = (int)value;
    else if (k == "ar_tma_stages" && (value == 2 || value == 3)) c->ar_tma_stages = (int)value;
    else if (k == "zero1_impl" && value >= 0 && value <= 2) c->zero1_impl = (int)value;
    else if (k == "ar_pipe_blocks" && value >= 1 && value <= kMaxBarrierBlocks) c->ar_pipe_blocks = (int)value;
    // cost decomposition only (tools/model_mode.py): the staged tap's copy-engine drain is not
    // issued, so the ring is never written -- restore and the host-ring fallback are invalid
    else if (k == "ablate_no_drain" && (value == 0 || value == 1) && c->no_shadow) c->ablate_no_drain = value;
    else return fail(c, CM_ERR_ARG, "unknown parameter %s=%lld", key, (long long)value);
    return CM_OK;
}

cm_status cm_timing(cm_ctx* c, int32_t enable, double* ms_out, int64_t* count_out) {
    if (!c) return CM_ERR_ARG;
    if (enable) {
        c->timing = true;
        c->timed.clear();
        c->ev_used = 0;
        memset(c->timed_bytes, 0, sizeof c->timed_bytes);
        return CM_OK;
    }
    memcpy(c->last_bytes, c->timed_bytes, sizeof c->last_bytes);
    c->timing = false;
    double ms[kTimingClasses] = {};
    int64_t cnt[kTimingClasses] = {};
    for (auto& t : c->timed) {
        CU(cudaEventSynchronize(t.second.second));
        float x = 0;
        CU(cudaEventElapsedTime(&x, t.second.first, t.second.second));
        ms[t.first] += x;
        cnt[t.first]++;
    }
    if (ms_out) memcpy(ms_out, ms, sizeof ms);
    if (count_out) memcpy(count_out, cnt, sizeof cnt);
    c->timed.clear();
    c->ev_used = 0;
    return CM_OK;
}

cm_status cm_barrier(cm_ctx* c, void* stream) {
    if (!c) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->connected) return fail(c, CM_ERR_STATE, "not connected");
    if (!c->barriers || c->n == 1) return CM_OK;   // virtual ranks: one stream orders them already
    barrier_kernel<<<1, 32, 0, S(stream)>>>(c->pads, c->n, c->rank, ++c->epoch);
    c->launches++;
    CHECK_LAUNCH();
    c->last_s = S(stream);
    c->last_kind = 0;
    return CM_OK;
}

cm_status cm_check(cm_ctx* c, int64_t* step, int64_t* index) {
    if (!c) return CM_ERR_ARG;
    const int64_t st = c->nf_host ? c->nf_host[0] : -1;
    const int64_t ix = c->nf_host ? c->nf_host[1] : -1;
    if (step) *step = st;
    if (index) *index = ix;
    return st >= 0 ? check_nf(c) : CM_OK;
}

cm_status cm_timing_bytes(const cm_ctx* c, int64_t* bytes_out) {
    if (!c || !bytes_out) return CM_ERR_ARG;
    memcpy(bytes_out, c->last_bytes, sizeof c->last_bytes);
    return CM_OK;
}

size_t cm_blob_size(void) { return sizeof(Blob); }

const char* cm_last_error(const cm_ctx* c) { return c ? c->err.c_str() : "null context"; }

cm_status cm_plan_buckets(const cm_layer_table* t, int32_t world_size, int64_t* out_padded,
                          int32_t* out_nb, int64_t* tensor_off) {
    if (!t || !t->numel || !out_padded || !out_nb) return CM_ERR_ARG;
    if (t->grad_dtype != CM_F32 && t->grad_dtype != CM_BF16) return CM_ERR_CONFIG;
    if (world_size < 1 || world_size > kMaxRanks) return CM_ERR_CONFIG;
    PlanOut po;
    if (!plan(t->numel, t->n_tensors, t->cap_bytes, t->grad_dtype == CM_F32 ? 4 : 2, world_size, po))
        return CM_ERR_CONFIG;
    *out_padded = po.total;
    *out_nb = (int32_t)po.buckets.size();
    if (tensor_off) memcpy(tensor_off, po.tensor_off.data(), sizeof(int64_t) * t->n_tensors);
    return CM_OK;
}

cm_status cm_plan_bucket_table(const cm_layer_table* t, int32_t world_size, int32_t capacity, int64_t* off,
                               int64_t* padded, int64_t* used, int32_t* out_n_buckets) {
    if (!t || !t->numel || !out_n_buckets) return CM_ERR_ARG;
    if (t->grad_dtype != CM_F32 && t->grad_dtype != CM_BF16) return CM_ERR_CONFIG;
    if (world_size < 1 || world_size > kMaxRanks) return CM_ERR_CONFIG;
    PlanOut po;
    if (!plan(t->numel, t->n_tensors, t->cap_bytes, t->grad_dtype == CM_F32 ? 4 : 2, world_size, po))
        return CM_ERR_CONFIG;
    *out_n_buckets = (int32_t)po.buckets.size();
    if ((int64_t)po.buckets.size() > (int64_t)capacity) return CM_ERR_ARG;
    for (size_t b = 0; b < po.buckets.size(); ++b) {
        if (off) off[b] = po.buckets[b].off;
        if (padded) padded[b] = po.buckets[b].padded;
        if (used) used[b] = po.buckets[b].used;
    }
    return CM_OK;
}

cm_status cm_init(const cm_config* cfg, cm_ctx** out) {
    if (!cfg || !out) return CM_ERR_ARG;
    *out = nullptr;
    if (cfg->world_size < 1 || cfg->world_size > kMaxRanks) return CM_ERR_CONFIG;
    if (cfg->rank < 0 || cfg->rank >= cfg->world_size) return CM_ERR_CONFIG;
    if (cfg->ring_depth < 2 || cfg->ring_depth > 64) return CM_ERR_CONFIG;
    if (cfg->shadow_place != CM_SHADOW_HOST && cfg->shadow_place != CM_SHADOW_DEVICE) return CM_ERR_CONFIG;
    if (cfg->persist_every < 0 || cfg->persist_every > cfg->ring_depth) return CM_ERR_CONFIG;
    const bool no_tap = (cfg->flags & CM_FLAG_NO_TAP) != 0;
    if (!no_tap && (!cfg->shm_name || !cfg->shm_name[0] || strlen(cfg->shm_name) > 200))
        return CM_ERR_CONFIG;
    cm_ctx* c = new cm_ctx();
    c->cfg = *cfg;
    c->shm_name = cfg->shm_name ? cfg->shm_name : "";
    c->cfg.shm_name = nullptr;
    c->n = cfg->world_size;
    c->rank = cfg->rank;
    c->dev = cfg->device;
    c->D = cfg->ring_depth;
    c->no_tap = no_tap;
    c->no_shadow = (cfg->flags & CM_FLAG_NO_SHADOW) != 0 && !no_tap;
    c->attach = (cfg->flags & CM_FLAG_ATTACH) != 0;
    c->ce_tap = (cfg->flags & CM_FLAG_TAP_COPYENGINE) != 0;
    // default tap = staged; CM_FLAG_TAP_DIRECT = kernel stores straight into the host ring
    c->staged_tap = (cfg->flags & CM_FLAG_TAP_DIRECT) == 0 && !c->ce_tap;
    c->zero1 = (cfg->flags & CM_FLAG_ZERO1) != 0;
    if (c->zero1 && (c->ce_tap || !c->staged_tap))
        return fail(c, CM_ERR_CONFIG, "CM_FLAG_ZERO1 needs the staged tap (no TAP_DIRECT / TAP_COPYENGINE)");
    c->shadow_place = cfg->shadow_place;
    // one-shot push kernel for buckets <= 2 MiB / n (measured crossover vs two-shot: 1 MiB
    // at n=2, 512 KiB at n=4; profiles/r01c_oneshot_sweep.md)
    c->oneshot_max = std::min<int64_t>(kOsSlotBytes, (2ll << 20) / c->n);
    c->K = cfg->persist_every <= 1 ? 1 : cfg->persist_every;
    if (c->shadow_place == CM_SHADOW_DEVICE) c->K = 1;
    *out = c;   // returned even on failure so cm_last_error works; caller finalizes

    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (c->dev < 0 || c->dev >= ndev) return fail(c, CM_ERR_CONFIG, "device %d not present (%d)", c->dev, ndev);
    CU(cudaSetDevice(c->dev));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, c->dev));
    if (prop.major < 10)
        return fail(c, CM_ERR_CONFIG, "device %d is sm_%d%d; libcm is built for sm_100a", c->dev, prop.major,
                    prop.minor);
    c->sms = prop.multiProcessorCount;
    // signal pad: 2 regions x kMaxBarrierBlocks x kMaxRanks epochs, zero = never signalled
    const size_t pad_bytes = (size_t)kPadRegions * kMaxBarrierBlocks * kMaxRanks * sizeof(uint32_t);
    CU(cudaMalloc(&c->pad, pad_bytes));
    CU(cudaMemset(c->pad, 0, pad_bytes));

    CU(cudaMalloc(&c->d_bad, sizeof(unsigned long long)));
    CU(cudaHostAlloc((void**)&c->ctl, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    c->ctl[0] = -1;
    c->ctl[1] = -1;
    c->nf_host = c->ctl;
    {
        int64_t* d = nullptr;
        CU(cudaHostGetDevicePointer((void**)&d, c->ctl, 0));
        c->nf_dev = d;
    }
    CU(cudaMalloc(&c->d_nf, sizeof(int64_t)));
    {
        const int64_t none = -1;
        CU(cudaMemcpy(c->d_nf, &none, sizeof none, cudaMemcpyHostToDevice));
    }
    for (int i = 0; i < c->D; ++i) {
        cudaEvent_t a, b;
        CU(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        c->ev_tap_done.push_back(a);
        c->ev_slot_free.push_back(b);
    }
    c->slot_sc.assign(c->D, StepRec{});
    c->slot_sc_step.assign(c->D, -1);
    return CM_OK;
}

cm_status cm_register_buckets(cm_ctx* c, const cm_layer_table* t, void* grad, float* p, float* m, float* v,
                              void* blob_out, size_t* blob_len) {
    if (!c) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (c->registered) return fail(c, CM_ERR_STATE, "already registered");
    if (!t || !t->numel || !grad || !p || !m || !v || !blob_out || !blob_len)
        return fail(c, CM_ERR_ARG, "null argument");
    if (((uintptr_t)grad | (uintptr_t)p | (uintptr_t)m | (uintptr_t)v) & 15)
        return fail(c, CM_ERR_ARG, "buffers must be 16-byte aligned");
    if (*blob_len < sizeof(Blob)) return fail(c, CM_ERR_ARG, "blob buffer too small");
    if (t->grad_dtype != CM_F32 && t->grad_dtype != CM_BF16) return fail(c, CM_ERR_CONFIG, "bad dtype");
    c->dtype = t->grad_dtype;
    c->es = c->dtype == CM_F32 ? 4 : 2;
    PlanOut po;
    if (!plan(t->numel, t->n_tensors, t->cap_bytes, c->es, c->n, po))
        return fail(c, CM_ERR_CONFIG, "invalid layer table (empty, non-positive sizes or cap)");
    if ((int64_t)po.buckets.size() > (1 << 20)) return fail(c, CM_ERR_CONFIG, "too many buckets");
    c->buckets = po.buckets;
    c->P_pad = po.total;
    c->shard_numel = po.total / c->n;
    c->numel.assign(t->numel, t->numel + t->n_tensors);
    c->cap_bytes = t->cap_bytes;
    c->layout_hash = layout_hash_of(c->numel, c->cap_bytes, c->dtype, c->n);
    c->grad = grad; c->p = p; c->m = m; c->v = v;
    CU(cudaSetDevice(c->dev));
    CU(cudaMalloc(&c->d_buckets, sizeof(BucketDev) * c->buckets.size()));
    CU(cudaMemcpy(c->d_buckets, c->buckets.data(), sizeof(BucketDev) * c->buckets.size(),
                  cudaMemcpyHostToDevice));
    // direct tap: the last block of a bucket's launch publishes its flag.  One counter per
    // bucket: launches of different buckets may overlap (PDL), launches of one bucket never do
    CU(cudaMalloc(&c->d_done_ctr, sizeof(unsigned long long) * c->buckets.size()));
    CU(cudaMemset(c->d_done_ctr, 0, sizeof(unsigned long long) * c->buckets.size()));
    c->done_total.assign(c->buckets.size(), 0);

    // launch geometry (identical on every rank: same GPU model, same plan)
    int occ = c->dtype == CM_F32 ? ar_occupancy<F32Tag>(c->n) : ar_occupancy<BF16Tag>(c->n);
    c->ar_blocks_max = std::min(c->sms * occ, kMaxBarrierBlocks);
    int aocc = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&aocc, adamw_kernel<F32Tag>, kAdamThreads, 0);
    c->adam_blocks = c->sms * std::max(aocc, 1);
    c->shadow_blocks = c->sms * 2;
    c->misc_blocks = c->sms * 4;
    c->tma_blocks = c->sms;     // one 192 KB-smem block per SM
    int zocc = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&zocc, adamw_zero1_kernel<F32Tag, 8>, 256, 0);
    c->zero1_blocks = std::min(c->sms * std::max(zocc, 1), kMaxBarrierBlocks);
    int ztocc = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ztocc, adamw_zero1_tma_kernel<F32Tag, 8>, kZ1TmaThreads, 0);
    c->zero1_tma_blocks = std::min(c->sms * std::max(ztocc, 1), kMaxBarrierBlocks);
    int wocc = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wocc, adamw_wt_kernel<F32Tag>, kAdamThreads, 0);
    c->wt_blocks = c->sms * std::max(wocc, 1);
    int wocc1 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wocc1, adamw_wt1_kernel<F32Tag>, kAdamThreads, 0);
    c->wt1_blocks = c->sms * std::max(wocc1, 1);
    CU(cudaFuncSetAttribute(adamw_tma_kernel<F32Tag>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kTmaStages * TmaTile<F32Tag>::kStageBytes));
    set_ar_tma_smem_all<F32Tag>();
    set_ar_tma_smem_all<BF16Tag>();
    CU(cudaGetLastError());
    CU(cudaFuncSetAttribute(adamw_tma_kernel<BF16Tag>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kTmaStages * TmaTile<BF16Tag>::kStageBytes));

    // exchange blob
    Blob b{};
    b.magic = kMagic;
    b.token = process_token();
    b.world_size = c->n;
    b.rank = c->rank;
    b.device = c->dev;
    b.dtype = c->dtype;
    b.layout_hash = c->layout_hash;
    b.padded_numel = c->P_pad;
    // one-shot inbox (peer-mapped like the signal pad; a token allocation when n == 1)
    const size_t inbox_bytes = c->n > 1 ? 2 * (size_t)c->n * kOsSlotBytes : 256;
    CU(cudaMalloc(&c->inbox, inbox_bytes));
    void* ptrs[6] = {grad, p, m, v, c->pad, c->inbox};
    PFN_getAddressRange getRange = nullptr;
    cudaDriverEntryPointQueryResult q;
    CU(cudaGetDriverEntryPoint("cuMemGetAddressRange", (void**)&getRange, cudaEnableDefault, &q));
    if (!getRange) return fail(c, CM_ERR_CUDA, "cuMemGetAddressRange unavailable");
    for (int k = 0; k < 6; ++k) {
        CUdeviceptr base = 0;
        size_t sz = 0;
        if (getRange(&base, &sz, (CUdeviceptr)ptrs[k]) != CUDA_SUCCESS)
            return fail(c, CM_ERR_ARG, "buffer %d is not a device allocation", k);
        b.base[k] = (uint64_t)base;
        b.offset[k] = (uint64_t)((char*)ptrs[k] - (char*)base);
        b.raw[k] = (uint64_t)ptrs[k];
        CU(cudaIpcGetMemHandle(&b.handle[k], (void*)base));
    }
    memcpy(blob_out, &b, sizeof b);
    *blob_len = sizeof b;
    c->registered = true;
    return CM_OK;
}

static cm_status open_peer(cm_ctx* c, const Blob& b, int k, void** out) {
    const uint64_t key = b.base[k] ^ (b.token * 0x9E3779B97F4A7C15ull);
    for (auto& e : c->opened)
        if (e.first == key) { *out = (char*)e.second + b.offset[k]; return CM_OK; }
    void* ptr = nullptr;
    CU(cudaIpcOpenMemHandle(&ptr, b.handle[k], cudaIpcMemLazyEnablePeerAccess));
    c->opened.push_back({key, ptr});
    *out = (char*)ptr + b.offset[k];
    return CM_OK;
}

static cm_status create_or_attach_segment(cm_ctx* c);

// ---------------------------------------------------------------- NVLS multicast inbox
// SURVEY 8 row f2.  Rank 0 creates a multicast object (CUDA VMM), exports it as a POSIX
// file descriptor and passes it to the peers over an abstract Unix socket (SCM_RIGHTS);
// every rank adds its device, binds its own physical inbox, and maps both the multicast
// address (pushes) and its own unicast address (reads).  The socket carries three
// rendezvous points: all devices added -> bind; all bound -> use.
namespace {
struct Drv {
    CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
    CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
    CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                          unsigned long long);
    CUresult (*mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
    CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
    CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*memRelease)(CUmemGenericAllocationHandle);
    CUresult (*memExport)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
    CUresult (*memImport)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
    CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*addrFree)(CUdeviceptr, size_t);
    CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*memUnmap)(CUdeviceptr, size_t);
    CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    CUresult (*devAttr)(int*, CUdevice_attribute, CUdevice);
    bool ok = false;
};
Drv& drv() {
    static Drv d = [] {
        Drv x{};
        cudaDriverEntryPointQueryResult q;
        bool ok = true;
        auto get = [&](const char* name, void** fn) {
            if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || !*fn) ok = false;
        };
        get("cuMulticastCreate", (void**)&x.mcCreate);
        get("cuMulticastAddDevice", (void**)&x.mcAddDevice);
        get("cuMulticastBindMem", (void**)&x.mcBindMem);
        get("cuMulticastGetGranularity", (void**)&x.mcGran);
        get("cuMulticastUnbind", (void**)&x.mcUnbind);
        get("cuMemCreate", (void**)&x.memCreate);
        get("cuMemRelease", (void**)&x.memRelease);
        get("cuMemExportToShareableHandle", (void**)&x.memExport);
        get("cuMemImportFromShareableHandle", (void**)&x.memImport);
        get("cuMemAddressReserve", (void**)&x.addrReserve);
        get("cuMemAddressFree", (void**)&x.addrFree);
        get("cuMemMap", (void**)&x.memMap);
        get("cuMemUnmap", (void**)&x.memUnmap);
        get("cuMemSetAccess", (void**)&x.setAccess);
        get("cuDeviceGetAttribute", (void**)&x.devAttr);
        x.ok = ok;
        return x;
    }();
    return d;
}

bool sock_send(int fd, const void* p, size_t n, int pass_fd = -1) {
    struct iovec io = {(void*)p, n};
    struct msghdr m = {};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    char cbuf[CMSG_SPACE(sizeof(int))] = {};
    if (pass_fd >= 0) {
        m.msg_control = cbuf;
        m.msg_controllen = sizeof cbuf;
        struct cmsghdr* h = CMSG_FIRSTHDR(&m);
        h->cmsg_level = SOL_SOCKET;
        h->cmsg_type = SCM_RIGHTS;
        h->cmsg_len = CMSG_LEN(sizeof(int));
        memcpy(CMSG_DATA(h), &pass_fd, sizeof(int));
    }
    return sendmsg(fd, &m, MSG_NOSIGNAL) == (ssize_t)n;
}

bool sock_recv(int fd, void* p, size_t n, int* got_fd = nullptr, int timeout_ms = 120000) {
    struct pollfd pf = {fd, POLLIN, 0};
    if (poll(&pf, 1, timeout_ms) != 1) return false;
    struct iovec io = {p, n};
    struct msghdr m = {};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    char cbuf[CMSG_SPACE(sizeof(int))] = {};
    m.msg_control = cbuf;
    m.msg_controllen = sizeof cbuf;
    if (recvmsg(fd, &m, MSG_WAITALL) != (ssize_t)n) return false;
    if (got_fd) {
        *got_fd = -1;
        for (struct cmsghdr* h = CMSG_FIRSTHDR(&m); h; h = CMSG_NXTHDR(&m, h))
            if (h->cmsg_level == SOL_SOCKET && h->cmsg_type == SCM_RIGHTS) memcpy(got_fd, CMSG_DATA(h), sizeof(int));
    }
    return true;
}
}  // namespace

#define DRV(call)                                                                               \
    do {                                                                                        \
        CUresult r_ = (call);                                                                   \
        if (r_ != CUDA_SUCCESS) { err = #call; code = (int)r_; goto out; }                     \
    } while (0)

static cm_status setup_nvls(cm_ctx* c, uint64_t job_token) {
    Drv& d = drv();
    if (!d.ok) return fail(c, CM_ERR_CONFIG, "CM_FLAG_NVLS: driver multicast entry points unavailable");
    int mc_ok = 0;
    d.devAttr(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, c->dev);
    if (!mc_ok) return fail(c, CM_ERR_CONFIG, "CM_FLAG_NVLS: device %d has no NVLink multicast", c->dev);
    const char* err = nullptr;
    int code = 0;
    int lfd = -1, fds[kMaxRanks] = {-1, -1, -1, -1, -1, -1, -1, -1}, mcfd = -1;
    char tok = 0;
    CUmulticastObjectProp mp = {};
    size_t gran = 0;
    struct sockaddr_un addr = {};
    addr.sun_family = AF_UNIX;
    // abstract name, unique per job (rank 0's process token) and layout
    const int nl = snprintf(addr.sun_path + 1, sizeof(addr.sun_path) - 1, "cmnvls.%016llx.%016llx",
                            (unsigned long long)job_token, (unsigned long long)c->layout_hash);
    const socklen_t alen = (socklen_t)(offsetof(struct sockaddr_un, sun_path) + 1 + nl);
    mp.numDevices = (unsigned)c->n;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = 2 * (size_t)c->n * kOsSlotBytes;
    DRV(d.mcGran(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
    c->mc_size = (mp.size + gran - 1) / gran * gran;
    mp.size = c->mc_size;
    if (c->rank == 0) {
        lfd = socket(AF_UNIX, SOCK_STREAM, 0);
        if (lfd < 0 || bind(lfd, (struct sockaddr*)&addr, alen) != 0 || listen(lfd, kMaxRanks) != 0) {
            err = "socket/bind/listen";
            goto out;
        }
        DRV(d.mcCreate(&c->mc_handle, &mp));
        DRV(d.memExport(&mcfd, c->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
        for (int k = 1; k < c->n; ++k) {
            struct pollfd pf = {lfd, POLLIN, 0};
            if (poll(&pf, 1, 120000) != 1) { err = "accept timeout"; goto out; }
            int a = accept(lfd, nullptr, nullptr);
            int32_t who = -1;
            if (a < 0 || !sock_recv(a, &who, sizeof who) || who < 1 || who >= c->n || fds[who] >= 0) {
                if (a >= 0) close(a);
                err = "bad peer";
                goto out;
            }
            fds[who] = a;
            if (!sock_send(a, &c->mc_size, sizeof c->mc_size, mcfd)) { err = "send fd"; goto out; }
        }
    } else {
        fds[0] = socket(AF_UNIX, SOCK_STREAM, 0);
        int tries = 0;
        while (connect(fds[0], (struct sockaddr*)&addr, alen) != 0) {
            if (++tries > 12000) { err = "connect to rank 0"; goto out; }
            usleep(10000);
        }
        int32_t me = c->rank;
        size_t sz = 0;
        if (!sock_send(fds[0], &me, sizeof me) || !sock_recv(fds[0], &sz, sizeof sz, &mcfd) || mcfd < 0 ||
            sz != c->mc_size) {
            err = "receive multicast handle";
            goto out;
        }
        DRV(d.memImport(&c->mc_handle, (void*)(uintptr_t)mcfd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    }
    DRV(d.mcAddDevice(c->mc_handle, (CUdevice)c->dev));
    // rendezvous 1: every device added before anyone binds memory; 2: every inbox bound
    for (int phase = 0; phase < 2; ++phase) {
        if (phase == 1) {
            CUmemAllocationProp ap = {};
            ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            ap.location.id = c->dev;
            ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;   // as the multicast object
            DRV(d.memCreate(&c->mc_phys, c->mc_size, &ap, 0));
            DRV(d.mcBindMem(c->mc_handle, 0, c->mc_phys, 0, c->mc_size, 0));
        }
        if (c->rank == 0) {
            for (int k = 1; k < c->n; ++k)
                if (!sock_recv(fds[k], &tok, 1)) { err = "rendezvous (peer)"; goto out; }
            for (int k = 1; k < c->n; ++k)
                if (!sock_send(fds[k], &tok, 1)) { err = "rendezvous (root)"; goto out; }
        } else if (!sock_send(fds[0], &tok, 1) || !sock_recv(fds[0], &tok, 1)) {
            err = "rendezvous";
            goto out;
        }
    }
    {
        CUmemAccessDesc ad = {};
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.location.id = c->dev;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        DRV(d.addrReserve(&c->mc_va, c->mc_size, gran, 0, 0));
        DRV(d.memMap(c->mc_va, c->mc_size, 0, c->mc_handle, 0));
        DRV(d.setAccess(c->mc_va, c->mc_size, &ad, 1));
        DRV(d.addrReserve(&c->uc_va, c->mc_size, gran, 0, 0));
        DRV(d.memMap(c->uc_va, c->mc_size, 0, c->mc_phys, 0));
        DRV(d.setAccess(c->uc_va, c->mc_size, &ad, 1));
    }
    c->nvls = true;
out:
    if (mcfd >= 0) close(mcfd);
    if (lfd >= 0) close(lfd);
    for (int k = 0; k < kMaxRanks; ++k)
        if (fds[k] >= 0) close(fds[k]);
    if (!c->nvls)
        return fail(c, CM_ERR_CONFIG, "CM_FLAG_NVLS setup failed at %s (CUresult %d, errno %d)", err ? err : "?",
                    code, errno);
    return CM_OK;
}
#undef DRV

cm_status cm_connect(cm_ctx* c, const void* blobs, size_t blob_len) {
    if (!c) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->registered) return fail(c, CM_ERR_STATE, "cm_register_buckets first");
    if (c->connected) return fail(c, CM_ERR_STATE, "already connected");
    if (!blobs || blob_len != sizeof(Blob)) return fail(c, CM_ERR_ARG, "bad blobs");
    CU(cudaSetDevice(c->dev));
    std::vector<Blob> B(c->n);
    memcpy(B.data(), blobs, sizeof(Blob) * c->n);
    bool all_local = true, same_dev = true;
    for (int k = 0; k < c->n; ++k) {
        if (B[k].magic != kMagic || B[k].world_size != c->n || B[k].rank != k)
            return fail(c, CM_ERR_CONFIG, "blob %d malformed or out of rank order", k);
        if (B[k].layout_hash != c->layout_hash || B[k].padded_numel != c->P_pad || B[k].dtype != c->dtype)
            return fail(c, CM_ERR_CONFIG, "rank %d registered a different layout", k);
        if (B[k].token != process_token()) all_local = false;
        if (B[k].device != c->dev) same_dev = false;
    }
    c->in_process = all_local;
    // ranks that share one device and one process are "virtual ranks": the caller issues
    // them on one stream in order, so no kernel ever waits for another and no barrier is
    // needed (B200_PROFILING.md: never spin across launches on one GPU).
    c->barriers = !(all_local && same_dev) && !c->force_no_barriers;
    // Hard-kill safety of a host shadow shared by several processes: restore needs one step
    // that every shard can still reach.  When a rank's iteration-t kernel runs, every peer's
    // ring already holds step t-1 (its staging half of t-2 was drained), so a peer may be stuck
    // as low as t-1 (or t-2 while this shard persists step t over its older half).  This shard
    // keeps that reachable only if its older snapshot is <= t-2 and the ring from it survives
    // the overwrite of step t+1-D: K >= 2 and D >= K + 1.  Virtual
    // ranks restore only after every stream is synchronised (all drains landed).
    if (c->barriers && c->n > 1 && !c->no_tap && !c->no_shadow && c->shadow_place == CM_SHADOW_HOST) {
        if (c->K < 2) c->K = 2;
        if (c->D < c->K + 1)
            return fail(c, CM_ERR_CONFIG,
                        "host shadow across processes needs ring_depth >= persist_every + 1 (D=%d, K=%d): a "
                        "hard kill could otherwise leave no step every shard can reach", c->D, c->K);
    }
    for (int k = 0; k < c->n; ++k) {
        void* ptr[6];
        if (k == c->rank) {
            for (int j = 0; j < 6; ++j) ptr[j] = (void*)B[k].raw[j];
        } else if (B[k].token == process_token()) {
            if (B[k].device != c->dev) {
                cudaError_t e = cudaDeviceEnablePeerAccess(B[k].device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return fail(c, CM_ERR_CONFIG, "no peer access %d->%d: %s", c->dev, B[k].device,
                                cudaGetErrorString(e));
                cudaGetLastError();
            }
            for (int j = 0; j < 6; ++j) ptr[j] = (void*)B[k].raw[j];
        } else {
            for (int j = 0; j < 6; ++j) {
                cm_status s = open_peer(c, B[k], j, &ptr[j]);
                if (s != CM_OK) return s;
            }
        }
        c->peer_grad[k] = (char*)ptr[0];
        c->peer_p[k] = (float*)ptr[1];
        c->peer_m[k] = (float*)ptr[2];
        c->peer_v[k] = (float*)ptr[3];
        c->pads.p[k] = (uint32_t*)ptr[4];
        c->peer_inbox[k] = (char*)ptr[5];
    }
    if ((c->cfg.flags & CM_FLAG_NVLS) && c->n > 1) {
        if (!c->barriers) return fail(c, CM_ERR_CONFIG, "CM_FLAG_NVLS needs one process per GPU");
        cm_status s = setup_nvls(c, B[0].token);
        if (s != CM_OK) return s;
    }
    if (!c->no_tap) {
        cm_status s = create_or_attach_segment(c);
        if (s != CM_OK) return s;
    }
    c->issued.assign(c->buckets.size(), 0);
    c->issued_count = 0;
    c->applied.assign(c->buckets.size(), 0);
    c->applied_count = 0;
    c->cur_iter = 0;
    c->train_step = 0;
    c->shadow_enq = 0;
    c->released_upto = 0;
    c->hh_step[0] = 0;
    c->hh_step[1] = -1;
    c->connected = true;
    return CM_OK;
}

static cm_status snapshot_state(cm_ctx* c, int half, cudaStream_t s) {
    // shard r of this rank's p/m/v -> shadow half `half` (shard-local), one kernel
    ShardCopyParams P{};
    P.src[0] = c->p; P.src[1] = c->m; P.src[2] = c->v;
    for (int a = 0; a < 3; ++a) P.dst[a][0] = c->sd[half][a];
    P.buckets = c->d_buckets;
    P.nb = (int)c->buckets.size();
    P.n = c->n;
    P.rank = c->rank;
    P.dir = 0;
    P.barriers = 0;
    P.mv_local = c->zero1 ? 1 : 0;
    P.shard_nvec = c->shard_numel / 4;
    int64_t want = (P.shard_nvec + 255) / 256;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, c->misc_blocks));
    shard_copy_kernel<<<grid, 256, 0, s>>>(P);
    c->launches++;
    CHECK_LAUNCH();
    return CM_OK;
}

// NUMA node of the GPU's PCIe root (sysfs), -1 if unknown or a single-node host.
static int gpu_numa_node(int dev) {
    char bus[64];
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) return -1;
    for (char* q = bus; *q; ++q) *q = (char)tolower((unsigned char)*q);
    char path[160];
    snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/numa_node", bus);
    FILE* f = fopen(path, "r");
    if (!f) return -1;
    int node = -1;
    if (fscanf(f, "%d", &node) != 1) node = -1;
    fclose(f);
    return node;
}

// Place the (not yet touched) host segment on one NUMA node, MPOL_PREFERRED: the tap drains
// and snapshot persists are DMA writes from the GPU, and on a two-socket host pages that
// first-touch put on the far socket cross the inter-socket link (tools/numa_probe.py).
// Preferred, not bound: a node short of memory falls back instead of failing.  Best effort.
static void bind_segment_numa(cm_ctx* c) {
    c->numa_used = -1;
    const int node = c->numa_req == -2 ? gpu_numa_node(c->dev) : c->numa_req;
    if (node < 0 || node >= 64) return;
    unsigned long mask = 1ul << node;
    const long MPOL_PREFERRED_ = 1;
    if (syscall(SYS_mbind, c->seg, c->seg_size, MPOL_PREFERRED_, &mask, 8 * sizeof mask + 1, 0) == 0)
        c->numa_used = node;
}

static cm_status create_or_attach_segment(cm_ctx* c) {
    char name[256];
    snprintf(name, sizeof name, "/%s.r%d", c->shm_name.c_str(), c->rank);
    const size_t nb = c->buckets.size();
    SegHeader h{};
    h.magic = kMagic;
    h.version = kVersion;
    h.world_size = c->n;
    h.rank = c->rank;
    h.dtype = c->dtype;
    h.ring_depth = c->D;
    h.n_buckets = (int32_t)nb;
    h.shadow_place = c->shadow_place;
    h.shard_numel = c->shard_numel;
    h.layout_hash = c->layout_hash;
    h.meta_off = kAlign;
    h.flags_off = align_up(h.meta_off + sizeof(SlotMeta) * c->D, kAlign);
    h.ring_off = align_up(h.flags_off + sizeof(uint64_t) * nb * c->D, kAlign);
    h.state_off = align_up(h.ring_off + (size_t)c->D * c->shard_numel * c->es, kAlign);
    const size_t state_bytes =
        (c->shadow_place == CM_SHADOW_HOST && !c->no_shadow) ? 6 * (size_t)c->shard_numel * 4 : 0;
    h.total = align_up(h.state_off + state_bytes, kAlign);

    if (c->attach) {
        c->shm_fd = shm_open(name, O_RDWR, 0600);
        if (c->shm_fd < 0) return fail(c, CM_ERR_STATE, "attach: no shadow segment %s", name);
        struct stat stt;
        fstat(c->shm_fd, &stt);
        if ((size_t)stt.st_size != h.total)
            return fail(c, CM_ERR_STATE, "attach: segment %s has size %zu, layout needs %zu", name,
                        (size_t)stt.st_size, (size_t)h.total);
    } else {
        // A surviving segment is the only restore source after a hard kill: never delete it
        // implicitly.  CM_FLAG_OVERWRITE states an intentional fresh start.
        if (c->cfg.flags & CM_FLAG_OVERWRITE) shm_unlink(name);
        c->shm_fd = shm_open(name, O_RDWR | O_CREAT | O_EXCL, 0600);
        if (c->shm_fd < 0 && errno == EEXIST)
            return fail(c, CM_ERR_STATE,
                        "shadow segment %s exists (a previous run's restore source): attach with CM_FLAG_ATTACH, "
                        "or start fresh with CM_FLAG_OVERWRITE / cm_unlink_shadow", name);
        if (c->shm_fd < 0) return fail(c, CM_ERR_CONFIG, "shm_open(%s) failed: %s", name, strerror(errno));
        if (ftruncate(c->shm_fd, (off_t)h.total) != 0)
            return fail(c, CM_ERR_CONFIG, "ftruncate(%s, %zu) failed: %s", name, (size_t)h.total, strerror(errno));
    }
    c->seg_size = h.total;
    void* mp = mmap(nullptr, c->seg_size, PROT_READ | PROT_WRITE, MAP_SHARED, c->shm_fd, 0);
    if (mp == MAP_FAILED) return fail(c, CM_ERR_CONFIG, "mmap(%s) failed: %s", name, strerror(errno));
    c->seg = (char*)mp;
    c->hdr = (SegHeader*)c->seg;
    if (!c->attach) bind_segment_numa(c);   // before the first touch (header write, pinning)
    if (c->attach) {
        const SegHeader& e = *c->hdr;
        if (e.magic != kMagic || e.version != kVersion || e.layout_hash != c->layout_hash ||
            e.world_size != c->n || e.rank != c->rank || e.ring_depth != c->D || e.dtype != c->dtype ||
            e.shard_numel != c->shard_numel || e.shadow_place != c->shadow_place || e.total != h.total)
            return fail(c, CM_ERR_STATE, "attach: segment %s layout differs from this context", name);
    } else {
        memcpy(c->seg, &h, sizeof h);
        c->hdr->shadow_step = -1;
        c->hdr->half_step[0] = -1;
        c->hdr->half_step[1] = -1;
        c->hdr->nf_step = -1;
        c->hdr->nf_index = -1;
        for (int i = 0; i < c->D; ++i) slot_meta(c, i)->step_tag = -1;
    }
    CU(cudaHostRegister(c->seg, c->seg_size, cudaHostRegisterMapped | cudaHostRegisterPortable));
    c->seg_registered = true;
    CU(cudaHostGetDevicePointer((void**)&c->seg_dev, c->seg, 0));
    c->nf_host = &c->hdr->nf_step;    // the report now survives the process (restore reads it)
    c->nf_dev = to_dev(c, &c->hdr->nf_step);
    {   // an attached segment may carry a previous run's report: the device word follows it
        const int64_t st = c->hdr->nf_step;
        CU(cudaMemcpy(c->d_nf, &st, sizeof st, cudaMemcpyHostToDevice));
    }
    if (c->no_shadow) return CM_OK;   // tap-only benchmark mode: ring + flags, no replica
    if (c->shadow_place == CM_SHADOW_HOST) {
        float* base = (float*)(c->seg + c->hdr->state_off);
        for (int hf = 0; hf < 2; ++hf)
            for (int a = 0; a < 3; ++a) c->sh[hf][a] = base + ((size_t)hf * 3 + a) * c->shard_numel;
    } else if (c->attach) {
        return fail(c, CM_ERR_STATE, "DEVICE-placed shadow cannot be attached after a restart");
    }
    CU(cudaMalloc(&c->state_dev_alloc, 6 * (size_t)c->shard_numel * 4));
    CU(cudaMemset(c->state_dev_alloc, 0, 6 * (size_t)c->shard_numel * 4));
    for (int hf = 0; hf < 2; ++hf)
        for (int a = 0; a < 3; ++a) c->sd[hf][a] = c->state_dev_alloc + ((size_t)hf * 3 + a) * c->shard_numel;
    if (!c->attach) {
        // reading R19: the shadow starts as a copy of the step-0 training state
        CU(cudaDeviceSynchronize());
        cm_status s = snapshot_state(c, 0, 0);
        if (s != CM_OK) return s;
        if (c->shadow_place == CM_SHADOW_HOST)
            for (int a = 0; a < 3; ++a)
                CU(cudaMemcpy(c->sh[0][a], c->sd[0][a], (size_t)c->shard_numel * 4, cudaMemcpyDeviceToHost));
        CU(cudaDeviceSynchronize());
        c->hdr->half_step[0] = 0;
        c->hdr->shadow_step = 0;
    }
    return CM_OK;
}

// Device -> host copy into the pinned, mapped segment on stream s: copy engine (full link
// rate), or with drain_ctas > 0 the low-intensity SM drain kernel (host pointer -> its
// device alias).  Both are stream-ordered like the other, so flags published after it on
// the same stream follow the data (posted writes stay ordered).
// Auto policy (drain_ctas = -1), from measurements (profiles/r01c_interference.md): a copy
// engine saturates the device->host link, which slows the GPU's launch-bound work, most when
// several GPUs share the host's root complex; an SM drain stores at ~11 GB/s per CTA without
// saturating it but holds SM slots.  Demand = per-step D2H (tap S/n + snapshot 12 L / K) over
// the measured step period.  Measured best (GPT-2 model mode, Llama-8B-shaped filler):
//   one GPU                        -> copy engine  (GPT-2: +2.2% vs NCCL; SM drains +5..+10%)
//   n > 1, demand <= 2.5 GB/s      -> 1 CTA        (GPT-2 n=4: +0.9%; copy engine +3.3%)
//   n > 1, demand  > 2.5 GB/s      -> 2 CTAs       (GPT-2 n=2: +1.6%, 1 CTA +3.3%;
//                                                   Llama n=4: -1.3% vs NCCL, copy engine +0.3%)
//   demand > 12.5 GB/s (little to hide under: the step is near link-bound) -> copy engine
// The step period is the GPU's (events after each step's optimizer kernel), not the host's:
// the host runs ahead of the GPU, and a host-side period once mixed a sync before a timed
// region into the estimate, sent the first iterations of a link-bound 2-GPU step to a 2-CTA
// SM drain that cannot keep up, and made that step measure 8.2 or 12-14 ms by chance.
constexpr double kSmDrainPerCta = 2.5e9;
constexpr int kSmDrainMaxCtas = 2;
// Above ~half the 2-CTA SM drain's ~25 GB/s the SM drain queues up and stalls the step:
// Llama-8B-shaped filler at n=4 (profiles/r01h_c4_sweep_n4.jsonl), T=8k tokens/GPU, 17 GB/s
// of demand on 2 CTAs: +3.8% vs NCCL; T=16k, 10 GB/s on 2 CTAs: -1.35%.
constexpr double kLinkBoundDemand = 12.5e9;
static int drain_ctas_now(const cm_ctx* c) {
    if (c->drain_ctas >= 0) return c->drain_ctas;
    if (c->n == 1 || c->iter_period_s <= 0.0) return 0;
    double bytes = (double)c->shard_numel * c->es;
    if (c->shadow_place == CM_SHADOW_HOST && !c->no_shadow) bytes += 12.0 * (double)c->shard_numel / c->K;
    const double demand = bytes / c->iter_period_s;
    if (demand > kLinkBoundDemand) return 0;
    return std::min(kSmDrainMaxCtas, std::max(1, (int)std::ceil(demand / kSmDrainPerCta)));
}

// cls: cm_timing class of the copy (5 tap drain, 6 snapshot persist)
static cm_status d2h(cm_ctx* c, char* host_dst, const void* dev_src, size_t bytes, cudaStream_t s, int cls) {
    TimedScope ts(c, cls, s);
    if (c->timing) c->timed_bytes[cls] += (int64_t)bytes;
    const int ctas = drain_ctas_now(c);
    if (ctas <= 0 || (bytes & 15) || ((uintptr_t)dev_src & 15) || ((uintptr_t)host_dst & 15)) {
        CU(cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, s));
        return CM_OK;
    }
    const int64_t nvec = (int64_t)(bytes / 16);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctas, (nvec + 255) / 256));
    drain_kernel<<<grid, 256, 0, s>>>((const uint4*)dev_src, (uint4*)to_dev(c, host_dst), nvec);
    c->launches++;
    CHECK_LAUNCH();
    return CM_OK;
}

// Issue the pending tap drain: one D2H of the run's contiguous source range into the ring.
// The iteration's tap flags are published once, after its last drain (restore can only use
// a slot whose every bucket is in, so per-bucket flags would buy nothing -- and a flag kernel
// between two copies idles the copy engine while its launch is fetched over the busy link).
// Small shards (Llama's norm buckets, the one-shot path) coalesce into one copy.
static cm_status flush_drain(cm_ctx* c, cudaStream_t s) {
    if (c->dr_b0 < 0) return CM_OK;
    CU(cudaEventRecord(c->ev_ar, s));
    CU(cudaStreamWaitEvent(c->cs_tap, c->ev_ar, 0));
    {
        cm_status st = d2h(c, c->dr_dst, c->dr_src, c->dr_bytes, c->cs_tap, 5);
        if (st != CM_OK) return st;
    }
    c->dr_b0 = c->dr_b1 = -1;
    c->dr_bytes = 0;
    return CM_OK;
}

cm_status cm_allreduce_multicast(cm_ctx* c, int32_t bucket, int64_t t, void* stream) {
    if (!c) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->connected) return fail(c, CM_ERR_STATE, "not connected");
    if (bucket < 0 || bucket >= (int32_t)c->buckets.size()) return fail(c, CM_ERR_ARG, "bucket %d out of range", bucket);
    cudaStream_t s = S(stream);
    if (t != c->cur_iter) {
        if (t == c->cur_iter + 1 && c->issued_count == (int)c->buckets.size()) {
            c->cur_iter = t;
            std::fill(c->issued.begin(), c->issued.end(), 0);
            c->issued_count = 0;
            std::fill(c->applied.begin(), c->applied.end(), 0);
            c->applied_count = 0;
        } else {
            return fail(c, CM_ERR_STATE, "iteration %lld out of order (current %lld, %d/%zu buckets issued)",
                        (long long)t, (long long)c->cur_iter, c->issued_count, c->buckets.size());
        }
    }
    if (c->issued[bucket]) return fail(c, CM_ERR_STATE, "bucket %d of iteration %lld issued twice", bucket, (long long)t);
    const int slot = (int)(t % c->D);
    if (c->no_tap && c->n == 1 && !c->zero1) {   // nothing to reduce, gather or tap
        c->issued[bucket] = 1;
        c->issued_count++;
        return CM_OK;
    }
    // n == 1 with the copy-engine tap: the reduced value is the local gradient, so no kernel
    // runs; only the copy engine moves the bucket to the ring (below)
    const bool skip_kernel = c->n == 1 && c->ce_tap && !c->no_tap;
    if (!c->no_tap && !c->no_shadow && c->issued_count == 0 && t >= c->D) {
        // lossless flow control: slot t mod D must have been consumed by the shadow's
        // step t-D+1 (backpressure, never drop or overwrite)
        if (c->released_upto < t - c->D + 1)
            return fail(c, CM_ERR_STATE,
                        "ring slot %d still holds iteration %lld: the shadow step (and, for a host shadow, "
                        "the snapshot) covering it was not enqueued (shadow at %lld, released < %lld)",
                        slot, (long long)(t - c->D), (long long)c->shadow_enq, (long long)c->released_upto);
        CU(cudaStreamWaitEvent(s, c->ev_slot_free[slot], 0));
    }
    const BucketDev& B = c->buckets[bucket];
    const int64_t shard = B.padded / c->n;
    ArParams P{};
    const int64_t byte_off = (B.off + (int64_t)c->rank * shard) * c->es;
    for (int k = 0; k < c->n; ++k) P.buf[k] = c->peer_grad[k] + byte_off;
    P.nvec = shard * c->es / 16;
    P.pads = c->pads;
    P.epoch = ++c->epoch;
    P.rank = c->rank;
    P.barriers = c->barriers ? 1 : 0;
    P.ag = (c->n > 1 && !c->zero1) ? 1 : 0;   // ZeRO-1 gathers the updated params instead
    // PDL (multi-process ranks or n == 1, cm_set_param "pdl"): wait for the predecessor only if it may
    // have touched this bucket, i.e. unless the previous launch of this context on `s` was
    // its all-reduce kernel of another bucket of the same iteration.  Never with exit
    // barriers: an exit barrier's ">=" could then be met by the NEXT launch's block of the
    // same index (its entry barrier is ordered by the trigger, its exit is not).
    const bool exit_barrier = !(c->lazy_exit || c->zero1);
    // n == 1 (no barriers): consecutive buckets' copies into staging overlap launch and ramp.
    // Not for virtual ranks: rank k+1's kernel reads the bucket rank k's all-gather rewrites.
    const bool pdl = (c->pdl || c->pdl_force) &&
                     ((c->barriers && (!exit_barrier || c->pdl_force)) || c->n == 1);
    P.pdl_wait = (pdl && c->last_s == s && c->last_kind == 1 && c->last_iter == t) ? 0 : 1;
    P.pdl_mode = c->pdl_mode;
    P.nf = c->nfref();                          // non-finite reduced values -> CM_ERR_INVARIANT
    P.elem0 = B.off + (int64_t)c->rank * shard;
    P.nf_step = t + 1;
    // exit barrier only when the training step does not fence the iteration: ZeRO-1's
    // optimizer ends in a barrier; the replicated AdamW starts with one when lazy_exit
    P.exit_barrier = exit_barrier ? 1 : 0;
    // tap modes: fused (kernel stores to the host ring), staged (kernel stores to an HBM
    // staging half, a copy engine drains it to the ring), copy-engine (CE reads the reduced
    // shard back from the grad buffer after the kernel)
    const bool fused_tap = !c->no_tap && !c->ce_tap && !c->staged_tap;
    // ZeRO-1 always reduces into the staging half: the sharded AdamW reads it from there
    const bool staged = (!c->no_tap && c->staged_tap) || c->zero1;
    if (staged) {
        if (!c->stage_buf[0]) {
            for (int i = 0; i < 2; ++i) {
                CU(cudaMalloc(&c->stage_buf[i], (size_t)c->shard_numel * c->es));
                CU(cudaEventCreateWithFlags(&c->ev_stage_free[i], cudaEventDisableTiming));
                CU(cudaEventCreateWithFlags(&c->ev_ar_done[i], cudaEventDisableTiming));
                CU(cudaEventCreateWithFlags(&c->ev_stage_consumed[i], cudaEventDisableTiming));
            }
        }
        if (c->issued_count == 0) {
            // staging half t&1 held iteration t-2: wait until it is drained to the ring and,
            // if the shadow step t-1 reads it from HBM, until that step has read it
            const int h = (int)(t & 1);
            CU(cudaStreamWaitEvent(s, c->ev_stage_free[h], 0));
            if (c->stage_consumer[h]) CU(cudaStreamWaitEvent(s, c->ev_stage_consumed[h], 0));
            c->stage_consumer[h] = false;
            c->stage_iter[h] = t;
        }
    }
    if (fused_tap) P.tap = ring_slot_dev(c, slot) + B.shard_off * c->es;
    else if (staged) P.tap = (char*)c->stage_buf[t & 1] + B.shard_off * c->es;
    const int64_t want = (P.nvec + (int64_t)kArThreads * kArUnroll - 1) / ((int64_t)kArThreads * kArUnroll);
    // grid: buckets up to ar_grid_switch_bytes take one block per SM (leaves room for the next
    // bucket's blocks to launch early under PDL; measured faster for 16-48 MiB, profiles/
    // r01t_arblocks_*), larger ones the co-resident cap of the n-rank instance
    int cap_blocks = (c->n == 1 && fused_tap) ? std::min(c->ar_blocks_tap_only, c->ar_blocks_max) : c->ar_blocks_max;
    if (c->n > 1 && c->ar_blocks_user == 0 && B.padded * c->es <= c->ar_grid_switch) cap_blocks = std::min(cap_blocks, c->sms);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, cap_blocks));
    if (fused_tap) {
        P.done_ctr = c->d_done_ctr + bucket;
        c->done_total[bucket] += (unsigned long long)grid;
        P.done_target = c->done_total[bucket];
        P.tap_flag = to_dev(c, slot_flags(c, slot) + bucket);
        P.tap_flag_value = (uint64_t)(t + 1);
    }
    // small buckets take the one-shot push kernel (multi-process ranks only:
    // virtual ranks share one stream, where a rank cannot wait for its peers' pushes;
    // they use the two-shot kernel, which computes the same rank-order sum)
    // (ZeRO-1: the push reduce-scatter variant -- shard k goes to rank k only, no all-gather;
    // the NVLS multicast push is for the all-reduce form only)
    const bool oneshot = c->n > 1 && c->barriers && B.padded * c->es <= c->oneshot_max;
    if (oneshot && !skip_kernel) {
        OsParams O{};
        const int64_t bucket_bytes = B.padded * c->es;
        const int h = (int)(P.epoch & 1);
        O.own = c->peer_grad[c->rank] + B.off * c->es;
        for (int k = 0; k < c->n; ++k) {
            O.push[k] = c->peer_inbox[k] + ((size_t)h * c->n + c->rank) * kOsSlotBytes;
            const char* in = c->nvls ? (const char*)c->uc_va : c->inbox;
            O.inbox[k] = in + ((size_t)h * c->n + k) * kOsSlotBytes;
        }
        if (c->nvls && !c->zero1) O.mc = (char*)c->mc_va + ((size_t)h * c->n + c->rank) * kOsSlotBytes;
        O.tap = P.tap;
        O.nvec = bucket_bytes / 16;
        O.shard_lo = (int64_t)c->rank * (shard * c->es / 16);
        O.shard_hi = O.shard_lo + shard * c->es / 16;
        O.shard_vec = shard * c->es / 16;
        O.rs_only = c->zero1 ? 1 : 0;
        O.pads = c->pads;
        O.epoch = P.epoch;
        O.rank = c->rank;
        O.nf = c->nfref();
        O.elem0 = B.off;
        O.nf_step = t + 1;
        const int og = (int)std::max<int64_t>(1, std::min<int64_t>((O.nvec + kOsThreads - 1) / kOsThreads,
                                                                   kMaxBarrierBlocks));
        if (fused_tap) {
            O.done_ctr = c->d_done_ctr + bucket;
            c->done_total[bucket] += (unsigned long long)og - (unsigned long long)grid;   // grid was counted above
            O.done_target = c->done_total[bucket];
            O.tap_flag = P.tap_flag;
            O.tap_flag_value = P.tap_flag_value;
        }
        TimedScope ts(c, 0, s);
        if (c->dtype == CM_F32) launch_os_t<F32Tag>(c->n, og, s, O);
        else launch_os_t<BF16Tag>(c->n, og, s, O);
        c->launches++;
        CHECK_LAUNCH();
    } else if (!skip_kernel && c->n == 1 && staged && !fused_tap && c->n1_ce_stage) {
        // n == 1: the reduced value is the local gradient, so the "all-reduce" is only the copy
        // of the bucket into the staging half; with "n1_copy_engine" a copy engine does it
        // (no SM time; the optimizer kernels still check every value for non-finites)
        TimedScope ts(c, 0, s);
        CU(cudaMemcpyAsync(P.tap, c->peer_grad[0] + byte_off, (size_t)shard * c->es, cudaMemcpyDeviceToDevice, s));
    } else if (!skip_kernel) {
        TimedScope ts(c, 0, s);
        const bool tma = c->n > 1 && !fused_tap &&
                         (c->ar_impl == 2 || (c->ar_impl == -1 && B.padded * c->es >= c->ar_tma_min));
        if (tma) {
            // bulk-copy pipeline: one block per SM over tiles of the shard
            P.tma_tile = ar_tma_tile(c);
            const int64_t tiles = (P.nvec * 16 + P.tma_tile - 1) / P.tma_tile;
            const int tg = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, c->sms));
            if (c->dtype == CM_F32) launch_ar_tma_t<F32Tag>(c->n, tg, s, P, pdl, c->ar_tma_stages);
            else launch_ar_tma_t<BF16Tag>(c->n, tg, s, P, pdl, c->ar_tma_stages);
        } else if (c->ar_impl == 1) {
            // one block per SM (co-resident by construction); the done counter of a direct
            // tap was advanced by `grid` above, re-base it on this grid
            const int pg = (int)std::max<int64_t>(1, std::min<int64_t>(
                (P.nvec + kArThreads - 1) / kArThreads, std::min(c->ar_pipe_blocks, c->sms)));
            if (fused_tap) {
                c->done_total[bucket] += (unsigned long long)pg - (unsigned long long)grid;
                P.done_target = c->done_total[bucket];
            }
            if (c->dtype == CM_F32) launch_ar_pipe_t<F32Tag>(c->n, pg, s, P);
            else launch_ar_pipe_t<BF16Tag>(c->n, pg, s, P);
        } else {
            if (c->dtype == CM_F32) launch_ar_t<F32Tag>(c->n, grid, s, P, pdl);
            else launch_ar_t<BF16Tag>(c->n, grid, s, P, pdl);
        }
        c->launches++;
        CHECK_LAUNCH();
    }
    if (!skip_kernel) {
        c->last_s = s;
        c->last_kind = 1;
        c->last_iter = t;
    }
    if (!c->no_tap && (c->ce_tap || staged) && !c->ablate_no_drain) {
        // copy-engine drain of the reduced shard to the host ring, decoupled from the training
        // stream: it overlaps the next buckets' all-reduce, the AdamW and (model mode) the
        // backward.  CE mode reads the grad buffer back (cm_apply_step then waits for these
        // copies before the caller may overwrite grads); staged mode reads the HBM staging
        // half the kernel wrote, so the grad buffer is free as soon as the kernel is done.
        if (!c->cs_tap) CU(cudaStreamCreateWithFlags(&c->cs_tap, cudaStreamNonBlocking));
        if (!c->ev_ar) CU(cudaEventCreateWithFlags(&c->ev_ar, cudaEventDisableTiming));
        const char* src = staged ? (const char*)c->stage_buf[t & 1] + B.shard_off * c->es
                                 : c->peer_grad[c->rank] + byte_off;
        char* dst = ring_slot_host(c, slot) + B.shard_off * c->es;
        const size_t bytes = (size_t)shard * c->es;
        // coalesce with the pending drain when this shard continues it (same iteration, next
        // bucket, contiguous source and destination); the pending run was launched before
        // this bucket's kernel, so the merged copy waits for both (stream order)
        const bool extend = c->dr_b0 >= 0 && c->dr_iter == t && bucket == c->dr_b1 + 1 &&
                            src == c->dr_src + c->dr_bytes && dst == c->dr_dst + c->dr_bytes &&
                            c->dr_bytes + bytes <= (size_t)kDrainCoalesce;
        if (!extend) {
            cm_status st = flush_drain(c, s);
            if (st != CM_OK) return st;
            c->dr_b0 = bucket;
            c->dr_iter = t;
            c->dr_src = src;
            c->dr_dst = dst;
        }
        c->dr_b1 = bucket;
        c->dr_bytes += bytes;
        // a run goes as soon as it is big enough to amortise a copy (small shards merge; the
        // link must not idle behind a long run); the iteration's last bucket flushes below
        if (c->dr_bytes >= (size_t)c->drain_flush) {
            cm_status st = flush_drain(c, s);
            if (st != CM_OK) return st;
        }
    }
    c->issued[bucket] = 1;
    c->issued_count++;
    if (c->issued_count == (int)c->buckets.size()) {
        cm_status st = flush_drain(c, s);
        if (st != CM_OK) return st;
        if (!c->no_tap && (c->ce_tap || staged) && !c->ablate_no_drain) {
            volatile uint64_t* fl = to_dev(c, slot_flags(c, slot));
            publish_range_kernel<<<1, 256, 0, c->cs_tap>>>(fl, (int)c->buckets.size(), (uint64_t)(t + 1));
            c->launches++;
            CHECK_LAUNCH();
        }
    }
    if (!c->no_tap && c->issued_count == (int)c->buckets.size()) {
        const bool via_ce = c->ce_tap || staged;
        CU(cudaEventRecord(c->ev_tap_done[slot], via_ce ? c->cs_tap : s));
        if (staged) {
            CU(cudaEventRecord(c->ev_stage_free[t & 1], c->cs_tap));
            CU(cudaEventRecord(c->ev_ar_done[t & 1], s));
        }
    }
    return CM_OK;
}

static cm_status step_checks(cm_ctx* c, int64_t step, int kind) {
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->connected) return fail(c, CM_ERR_STATE, "not connected");
    if (step != c->train_step + 1) return fail(c, CM_ERR_STATE, "step %lld follows %lld", (long long)step, (long long)c->train_step);
    if (c->cur_iter != step - 1 || c->issued_count != (int)c->buckets.size())
        return fail(c, CM_ERR_STATE, "step %lld before all buckets of iteration %lld were all-reduced (%d/%zu)",
                    (long long)step, (long long)(step - 1), c->issued_count, c->buckets.size());
    if (c->opt_kind >= 0 && c->opt_kind != kind)
        return fail(c, CM_ERR_STATE, "optimizer changed mid-run (%s after %s steps): m/v would change meaning",
                    kind == kOptSgd ? "SGD" : "AdamW", c->opt_kind == kOptSgd ? "SGD" : "AdamW");
    return CM_OK;
}

static cm_status apply_impl(cm_ctx* c, int64_t step, const StepRec& rec, void* stream);

cm_status cm_apply_step(cm_ctx* c, int64_t step, const cm_adamw* hp, void* stream) {
    if (!c || !hp) return CM_ERR_ARG;
    cm_status st = step_checks(c, step, kOptAdamW);
    if (st != CM_OK) return st;
    StepRec r;
    r.kind = kOptAdamW;
    r.a = make_scalars(c, step, *hp);
    return apply_impl(c, step, r, stream);
}

cm_status cm_apply_step_sgd(cm_ctx* c, int64_t step, const cm_sgd* hp, void* stream) {
    if (!c || !hp) return CM_ERR_ARG;
    cm_status st = step_checks(c, step, kOptSgd);
    if (st != CM_OK) return st;
    StepRec r;
    r.kind = kOptSgd;
    r.q = make_sgd_scalars(c, *hp);
    return apply_impl(c, step, r, stream);
}

// GPU period between consecutive training steps: the newest pair of step events (recorded
// after each step's optimizer kernel on the training stream) that have both completed and
// were not used yet.  Nothing completed yet (the host runs ahead): the estimate stands.
// One long interval (a pause for evaluation, a sync) counts at most 4x the estimate.
static void update_gpu_period(cm_ctx* c, int64_t step) {
    constexpr int E = cm_ctx::kStepEv;
    for (int64_t k = step - 1; k >= 2 && k > c->gper_last && k > step - E; --k) {
        const int a = (int)((k - 1) % E), b = (int)(k % E);
        if (c->ev_gstep_step[a] != k - 1 || c->ev_gstep_step[b] != k) continue;
        if (cudaEventQuery(c->ev_gstep[b]) != cudaSuccess) continue;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->ev_gstep[a], c->ev_gstep[b]) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        double dt = ms * 1e-3;
        if (c->iter_period_s > 0.0) dt = std::min(dt, 4.0 * c->iter_period_s);
        c->iter_period_s = c->iter_period_s > 0.0 ? 0.8 * c->iter_period_s + 0.2 * dt : dt;
        c->gper_last = k;
        return;
    }
}

// The optimizer step of ONE bucket (f1, cm_apply_bucket): the same element arithmetic over
// the bucket's elements (ZeRO-1: its shard, fused with the parameter all-gather), started by
// a per-bucket fence (block j waits for block j of every rank, i.e. for every rank's
// all-reduce kernel of this bucket to have finished: its all-gather stores landed here and
// nobody reads this bucket of our gradients any more).  No scalar record (cm_apply_step
// writes it once all buckets are done).
static cm_status launch_bucket_opt(cm_ctx* c, int b, int64_t step, const StepRec& rec, cudaStream_t s) {
    const BucketDev& B = c->buckets[b];
    AdamParams P{};
    set_step(P, rec);
    P.step = step;
    P.nf = c->nfref();
    if (c->zero1) {
        Zero1Params Z{};
        Z.g = (const char*)c->stage_buf[(step - 1) & 1] + B.shard_off * c->es;
        Z.j0 = B.shard_off;
        Z.L = B.padded / c->n;
        Z.m = c->m; Z.v = c->v;
        for (int k = 0; k < c->n; ++k) Z.p[k] = c->peer_p[k];
        Z.buckets = c->d_buckets;
        Z.nb = (int)c->buckets.size();
        Z.n = c->n; Z.rank = c->rank; Z.barriers = c->barriers ? 1 : 0;
        Z.s = P.s;
        Z.q = P.q;
        Z.pads = c->pads;
        Z.epoch = ++c->epoch;
        Z.step = step;
        Z.unroll2 = c->zero1_impl == 0 ? 0 : 1;
        Z.nf = c->nfref();
        Z.rec_kind = P.rec_kind;
        const int64_t want = (Z.L / 4 + 255) / 256;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, c->zero1_blocks));
        TimedScope ts(c, 1, s);
        if (Z.rec_kind == kOptSgd) {
            if (c->dtype == CM_F32) launch_zero1_t<F32Tag, kOptSgd>(c->n, grid, s, Z);
            else launch_zero1_t<BF16Tag, kOptSgd>(c->n, grid, s, Z);
        } else {
            if (c->dtype == CM_F32) launch_zero1_t<F32Tag, kOptAdamW>(c->n, grid, s, Z);
            else launch_zero1_t<BF16Tag, kOptAdamW>(c->n, grid, s, Z);
        }
        c->launches++;
        CHECK_LAUNCH();
        return CM_OK;
    }
    P.g = (const char*)c->grad + B.off * c->es;
    P.p_in = P.p_out = c->p + B.off;
    P.m_in = P.m_out = c->m + B.off;
    P.v_in = P.v_out = c->v + B.off;
    P.n = B.padded;
    P.nf_base = B.off;
    if (c->barriers && c->n > 1) {
        P.pads = c->pads;
        P.epoch = ++c->epoch;
        P.fence_n = c->n;
        P.fence_rank = c->rank;
    }
    TimedScope ts(c, 1, s);
    return launch_adamw(c, P, c->adam_blocks, s);
}

static bool same_rec(const StepRec& a, const StepRec& b) {
    float fa[10], fb[10];
    a.to_floats(fa);
    b.to_floats(fb);
    return a.kind == b.kind && memcmp(fa, fb, sizeof fa) == 0;
}

static cm_status apply_bucket_impl(cm_ctx* c, int32_t b, int64_t step, const StepRec& rec, void* stream) {
    if (b < 0 || b >= (int32_t)c->buckets.size()) return fail(c, CM_ERR_ARG, "bucket %d out of range", b);
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->connected) return fail(c, CM_ERR_STATE, "not connected");
    if (step != c->train_step + 1 || c->cur_iter != step - 1)
        return fail(c, CM_ERR_STATE, "bucket step %lld: training is at step %lld, iteration %lld", (long long)step,
                    (long long)c->train_step, (long long)c->cur_iter);
    if (!c->issued[b]) return fail(c, CM_ERR_STATE, "bucket %d of iteration %lld not all-reduced yet", b, (long long)(step - 1));
    if (c->applied[b]) return fail(c, CM_ERR_STATE, "bucket %d of step %lld applied twice", b, (long long)step);
    if (c->opt_kind >= 0 && c->opt_kind != rec.kind) return fail(c, CM_ERR_STATE, "optimizer changed mid-run");
    if (c->applied_count > 0 && !same_rec(rec, c->bucket_rec))
        return fail(c, CM_ERR_STATE, "bucket %d of step %lld: hyper-parameters differ from the step's first bucket", b,
                    (long long)step);
    cm_status st = launch_bucket_opt(c, b, step, rec, S(stream));
    if (st != CM_OK) return st;
    c->bucket_rec = rec;
    c->applied[b] = 1;
    c->applied_count++;
    c->last_s = S(stream);
    c->last_kind = 0;
    return CM_OK;
}

static cm_status apply_impl(cm_ctx* c, int64_t step, const StepRec& rec, void* stream) {
    if (c->applied_count > 0 && !same_rec(rec, c->bucket_rec))
        return fail(c, CM_ERR_STATE, "step %lld: hyper-parameters differ from its per-bucket steps", (long long)step);
    update_gpu_period(c, step);
    const int slot = (int)((step - 1) % c->D);
    c->slot_sc[slot] = rec;
    c->slot_sc_step[slot] = step;
    AdamParams P{};
    P.g = c->grad;
    P.p_in = c->p; P.m_in = c->m; P.v_in = c->v;
    P.p_out = c->p; P.m_out = c->m; P.v_out = c->v;
    P.n = c->P_pad;
    set_step(P, rec);
    P.step = step;
    P.nf = c->nfref();       // non-finite updated state -> CM_ERR_INVARIANT
    P.nf_base = 0;
    if (!c->no_tap) {
        SlotMeta* sm = slot_meta(c, slot);
        P.hp_rec = to_dev(c, sm->sc);
        P.hp_kind = to_dev(c, &sm->kind);
        P.hp_tag = to_dev(c, &sm->step_tag);
        P.step = step;
    }
    cm_status st;
    if (c->applied_count > 0) {
        // per-bucket steps already ran for some buckets (f1): the rest now, then the record
        for (int b = 0; b < (int)c->buckets.size(); ++b) {
            if (c->applied[b]) continue;
            st = launch_bucket_opt(c, b, step, rec, S(stream));
            if (st != CM_OK) return st;
            c->applied[b] = 1;
            c->applied_count++;
        }
        if (P.hp_rec) {
            record_kernel<<<1, 1, 0, S(stream)>>>(P);
            c->launches++;
            CHECK_LAUNCH();
        }
        st = CM_OK;
    } else if (c->zero1) {
        // ZeRO-1: AdamW on this rank's shard (reduced grads in staging half (step-1)&1),
        // fused with the NVLink all-gather of the updated parameters
        Zero1Params Z{};
        Z.g = c->stage_buf[(step - 1) & 1];
        Z.m = c->m; Z.v = c->v;
        for (int k = 0; k < c->n; ++k) Z.p[k] = c->peer_p[k];
        Z.buckets = c->d_buckets;
        Z.nb = (int)c->buckets.size();
        Z.n = c->n; Z.rank = c->rank; Z.barriers = c->barriers ? 1 : 0;
        Z.L = c->shard_numel;
        Z.s = P.s;
        Z.q = P.q;
        Z.pads = c->pads;
        Z.epoch = ++c->epoch;
        Z.hp_rec = P.hp_rec; Z.hp_kind = P.hp_kind; Z.hp_tag = P.hp_tag; Z.step = step;
        Z.unroll2 = c->zero1_impl;
        Z.nf = c->nfref();
        memcpy(Z.rec, P.rec, sizeof Z.rec);
        Z.rec_kind = P.rec_kind;
        const int64_t want = (Z.L / 4 + 255) / 256;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, c->zero1_blocks));
        {
            TimedScope ts(c, 1, S(stream));
            launch_zero1(c, Z, grid, S(stream));
        }
        c->launches++;
        cudaError_t e = cudaGetLastError();
        st = e == cudaSuccess ? CM_OK : fail(c, CM_ERR_CUDA, "zero1 launch: %s", cudaGetErrorString(e));
    } else {
        if (c->barriers && c->n > 1 && c->lazy_exit) {
            P.pads = c->pads;
            P.epoch = ++c->epoch;
            P.fence_n = c->n;
            P.fence_rank = c->rank;
        }
        TimedScope ts(c, 1, S(stream));
        st = launch_adamw(c, P, c->adam_blocks, S(stream));
    }
    if (st != CM_OK) return st;
    c->last_s = S(stream);
    c->last_kind = 0;
    {   // the GPU step clock of the drain policy
        const int k = (int)(step % cm_ctx::kStepEv);
        if (!c->ev_gstep[k]) CU(cudaEventCreate(&c->ev_gstep[k]));
        CU(cudaEventRecord(c->ev_gstep[k], S(stream)));
        c->ev_gstep_step[k] = step;
    }
    if (!c->no_tap && c->ce_tap)   // the caller may overwrite grads after this: taps first
        CU(cudaStreamWaitEvent(S(stream), c->ev_tap_done[slot], 0));
    c->train_step = step;
    c->grads_step = step;
    c->opt_kind = rec.kind;
    return CM_OK;
}

cm_status cm_apply_bucket(cm_ctx* c, int32_t bucket, int64_t step, const cm_adamw* hp, void* stream) {
    if (!c || !hp) return CM_ERR_ARG;
    StepRec r;
    r.kind = kOptAdamW;
    r.a = make_scalars(c, step, *hp);
    return apply_bucket_impl(c, bucket, step, r, stream);
}

cm_status cm_apply_bucket_sgd(cm_ctx* c, int32_t bucket, int64_t step, const cm_sgd* hp, void* stream) {
    if (!c || !hp) return CM_ERR_ARG;
    StepRec r;
    r.kind = kOptSgd;
    r.q = make_sgd_scalars(c, *hp);
    return apply_bucket_impl(c, bucket, step, r, stream);
}

// Shadow step s on rank r's shard (shard-local arrays of L elements).  Chunks of
// kStageElems elements pipeline through kStages staging buffers:
//   copy engine H2D : ring slot (s-1) mod D (host) -> staging          (sizeof(G) B/elem)
//   AdamW kernel    : HBM half (s-1)&1 -> HBM half s&1                 (28/26 B/elem HBM)
//   copy engine D2H : HBM half s&1 -> host half s&1 (HOST placement)   (12 B/elem)
// then the step is published in the segment header.  No SM ever waits on PCIe latency
// (an SM zero-copy variant measured 15 GB/s); the host link carries only the bytes that
// must persist.
static cm_status ensure_staging(cm_ctx* c) {
    if (c->stg_ready) return CM_OK;
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&c->cs_h2d, cudaStreamNonBlocking, lo));   // lo = least priority
    CU(cudaStreamCreateWithPriority(&c->cs_d2h, cudaStreamNonBlocking, lo));
    CU(cudaStreamCreateWithPriority(&c->cs_k, cudaStreamNonBlocking, lo));
    c->stg_elems = std::min<int64_t>(kStageElems, std::max<int64_t>(c->shard_numel, 8));
    for (int j = 0; j < kStages; ++j) {
        CU(cudaMalloc(&c->stg_g[j], (size_t)c->stg_elems * c->es));
        CU(cudaEventCreateWithFlags(&c->ev_stg_free[j], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->ev_stg_ready[j], cudaEventDisableTiming));
    }
    CU(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    c->stg_ready = true;
    return CM_OK;
}

// The queue of snapshot persists: their own low-priority stream (default), or with
// "persist_queue" = 1 the tap-drain stream, so drains and persists take the device->host link
// one at a time in issue order instead of splitting it.
static cudaStream_t persist_q(cm_ctx* c) {
    if (c->persist_on_tap && c->cs_tap) return c->cs_tap;
    return c->cs_d2h;
}

// One shadow step; returns (via *persisted) whether a host snapshot was written.  HBM
// half step&1 receives the new state.  HOST placement persists it to the older host half
// when step % K == 0 (or when forced): the host then holds a snapshot plus the tapped
// gradients since it -- every step remains recoverable from host memory alone (restore
// rolls forward over the ring), with 12/K instead of 12 bytes per element of D2H.
static cm_status shadow_step_enqueue(cm_ctx* c, int64_t step, const StepRec& rec, cudaStream_t s,
                                     bool force_persist, bool* persisted, const char* dev_g = nullptr,
                                     cudaEvent_t grads_consumed = nullptr) {
    const int slot = (int)((step - 1) % c->D);
    const int hin = (int)((step - 1) & 1), hout = (int)(step & 1);
    cm_status st = ensure_staging(c);
    if (st != CM_OK) return st;
    const bool host = c->shadow_place == CM_SHADOW_HOST;
    const bool persist = host && (force_persist || step % c->K == 0);
    const int ph = c->hh_step[0] <= c->hh_step[1] ? 0 : 1;     // overwrite the older snapshot
    volatile int64_t* hs = &c->hdr->half_step[host ? ph : hout];
    if (!host || persist) {
        st = publish(c, hs, -1, s);   // the half being rewritten is invalid until done
        if (st != CM_OK) return st;
    }
    const char* ring = ring_slot_host(c, slot);
    {
        CU(cudaEventRecord(c->ev_fork, s));
        CU(cudaStreamWaitEvent(c->cs_h2d, c->ev_fork, 0));
        CU(cudaStreamWaitEvent(c->cs_k, c->ev_fork, 0));
        CU(cudaStreamWaitEvent(c->cs_d2h, c->ev_fork, 0));
        // chunks pipeline the H2D (ring fallback) or the D2H persist with the kernels; with
        // the gradients already in HBM and nothing to persist, one launch covers the shard
        const int64_t L = c->shard_numel;
        const int64_t C = (dev_g && !persist) ? std::max<int64_t>(L, 1) : c->stg_elems;
        for (int64_t lo = 0, i = 0; lo < L; lo += C, ++i) {
            const int j = (int)(i % kStages);
            const int64_t len = std::min(C, L - lo);
            if (!dev_g) {
                // copy engine H2D of the ring chunk into staging j (once the kernel that used
                // staging j kStages chunks ago is done)
                CU(cudaStreamWaitEvent(c->cs_h2d, c->ev_stg_free[j], 0));
                CU(cudaMemcpyAsync(c->stg_g[j], ring + lo * c->es, (size_t)len * c->es, cudaMemcpyHostToDevice,
                                   c->cs_h2d));
                CU(cudaEventRecord(c->ev_stg_ready[j], c->cs_h2d));
                // AdamW on its own stream: a kernel delayed by busy SMs does not stall the copies
                CU(cudaStreamWaitEvent(c->cs_k, c->ev_stg_ready[j], 0));
            }
            AdamParams P{};
            P.g = dev_g ? (const void*)(dev_g + lo * c->es) : (const void*)c->stg_g[j];
            P.n = len;
            set_step(P, rec);
            P.p_in = c->sd[hin][0] + lo; P.m_in = c->sd[hin][1] + lo; P.v_in = c->sd[hin][2] + lo;
            P.p_out = c->sd[hout][0] + lo; P.m_out = c->sd[hout][1] + lo; P.v_out = c->sd[hout][2] + lo;
            P.step = step;
            P.nf = c->nfref();       // the shadow checks its own results too (index unknown: -1)
            P.nf_base = -1;
            P.skip_nf = c->d_nf;    // and never applies a flagged step (device word)
            {   // cm_timing class 2: the shadow's optimizer kernel itself, on its stream, after
                // its waits (the step's other parts -- persists -- are class 6)
                TimedScope ts(c, 2, c->cs_k);
                st = launch_adamw(c, P, c->shadow_blocks, c->cs_k);
            }
            if (st != CM_OK) return st;
            CU(cudaEventRecord(c->ev_stg_free[j], c->cs_k));
            if (persist) {   // copy engine D2H of the new state chunk into the host snapshot half
                cudaStream_t pq = persist_q(c);
                CU(cudaStreamWaitEvent(pq, c->ev_stg_free[j], 0));
                // SGD leaves v untouched (all zero in every half): p and the velocity only
                for (int k = 0; k < (rec.kind == kOptSgd ? 2 : 3); ++k)
                {
                    cm_status pst = d2h(c, (char*)(c->sh[ph][k] + lo), c->sd[hout][k] + lo, (size_t)len * 4, pq, 6);
                    if (pst != CM_OK) return pst;
                }
            }
        }
        CU(cudaEventRecord(c->ev_join, c->cs_k));
        // the gradients (HBM staging half) are consumed once the kernels are done: the
        // training stream may reuse the half without waiting for a snapshot persist
        if (grads_consumed) CU(cudaEventRecord(grads_consumed, c->cs_k));
        CU(cudaStreamWaitEvent(s, c->ev_join, 0));
        if (persist) {
            CU(cudaEventRecord(c->ev_join, persist_q(c)));
            CU(cudaStreamWaitEvent(s, c->ev_join, 0));
        }
    }
    if (!host || persist) {
        st = publish(c, hs, step, s, step);   // not if the step was flagged non-finite
        if (st != CM_OK) return st;
    }
    if (persist) c->hh_step[ph] = step;
    if (persisted) *persisted = persist;
    return publish(c, &c->hdr->shadow_step, step, s, step);
}

cm_status cm_shadow_apply(cm_ctx* c, int64_t step, void* side_stream) {
    if (!c) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->connected) return fail(c, CM_ERR_STATE, "not connected");
    if (c->no_tap || c->no_shadow) return fail(c, CM_ERR_STATE, "context has no shadow (CM_FLAG_NO_TAP/NO_SHADOW)");
    if (step != c->shadow_enq + 1)
        return fail(c, CM_ERR_STATE, "shadow step %lld after %lld: iteration gap", (long long)step, (long long)c->shadow_enq);
    const int slot = (int)((step - 1) % c->D);
    if (c->train_step < step || c->slot_sc_step[slot] != step)
        return fail(c, CM_ERR_STATE, "shadow step %lld before cm_apply_step(%lld)", (long long)step, (long long)step);
    cudaStream_t s = S(side_stream);
    // the shadow reads iteration step-1's reduced gradients from the HBM staging half the
    // tap wrote (no host-link traffic), unless that half was already reused (the shadow fell
    // more than one iteration behind): then from the host ring (copy-engine H2D)
    const int64_t it = step - 1;
    const int h = (int)(it & 1);
    const bool from_stage = c->staged_tap && c->stage_buf[h] && c->stage_iter[h] == it;
    if (from_stage) CU(cudaStreamWaitEvent(s, c->ev_ar_done[h], 0));
    if (c->shadow_after_train) {   // ablation: start after the training step's optimizer kernel
        const int k = (int)(step % cm_ctx::kStepEv);
        if (c->ev_gstep[k] && c->ev_gstep_step[k] == step) CU(cudaStreamWaitEvent(s, c->ev_gstep[k], 0));
    }
    else CU(cudaStreamWaitEvent(s, c->ev_tap_done[slot], 0));   // all taps of iteration step-1
    bool persisted = false;
    cm_status st = shadow_step_enqueue(c, step, c->slot_sc[slot], s, false, &persisted,
                                       from_stage ? (const char*)c->stage_buf[h] : nullptr,
                                       from_stage ? c->ev_stage_consumed[h] : nullptr);
    if (st != CM_OK) return st;
    if (from_stage) c->stage_consumer[h] = true;
    c->last_s = s;
    c->last_kind = 0;
    // release ring slots: DEVICE placement once consumed; HOST placement once a persisted
    // snapshot covers them (the ring is the log that makes every step recoverable)
    if (c->shadow_place == CM_SHADOW_DEVICE || persisted) {
        for (int64_t u = c->released_upto; u <= step - 1; ++u)
            CU(cudaEventRecord(c->ev_slot_free[u % c->D], s));
        c->released_upto = step;
    }
    c->shadow_enq = step;
    return CM_OK;
}

cm_status cm_gen_grads(cm_ctx* c, uint64_t seed, int64_t t, int32_t scale, void* stream) {
    if (!c) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->registered) return fail(c, CM_ERR_STATE, "not registered");
    const uint64_t K = [&] {
        uint64_t x = seed ^ ((uint64_t)c->rank << 48) ^ (uint64_t)t;
        uint64_t z = x + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }();
    const int64_t nvec = c->P_pad * c->es / 16;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nvec + 255) / 256, c->misc_blocks));
    TimedScope ts(c, 3, S(stream));
    if (c->dtype == CM_F32)
        gen_grads_kernel<F32Tag><<<grid, 256, 0, S(stream)>>>(c->grad, nvec, c->d_buckets, (int)c->buckets.size(), K, scale);
    else
        gen_grads_kernel<BF16Tag><<<grid, 256, 0, S(stream)>>>(c->grad, nvec, c->d_buckets, (int)c->buckets.size(), K, scale);
    c->launches++;
    c->last_s = S(stream);
    c->last_kind = 0;
    CHECK_LAUNCH();
    return CM_OK;
}

cm_status cm_init_state(cm_ctx* c, uint64_t seed, void* stream) {
    if (!c) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->registered) return fail(c, CM_ERR_STATE, "not registered");
    const uint64_t K = [&] {
        uint64_t x = seed ^ ((uint64_t)0xFFFF << 48) ^ 0ull;
        uint64_t z = x + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }();
    const int64_t nvec = c->P_pad / 4;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nvec + 255) / 256, c->misc_blocks));
    init_state_kernel<<<grid, 256, 0, S(stream)>>>(c->p, c->zero1 ? nullptr : c->m, c->zero1 ? nullptr : c->v, nvec,
                                                   c->d_buckets, (int)c->buckets.size(), K);
    if (c->zero1) {
        CU(cudaMemsetAsync(c->m, 0, (size_t)c->shard_numel * 4, S(stream)));
        CU(cudaMemsetAsync(c->v, 0, (size_t)c->shard_numel * 4, S(stream)));
    }
    c->launches++;
    c->last_s = S(stream);
    c->last_kind = 0;
    CHECK_LAUNCH();
    return CM_OK;
}

static cm_status verify_host_log(cm_ctx* c, int64_t T, cudaStream_t s, int64_t* gap_from);
static bool slot_complete(const char* base, const SegHeader* h, int D, int nb, int64_t s);

// Bitwise checks of the checkpoint against the training replica (PAPER.md:605,
// SPEC.md:588-596).  See cm.h for the scopes.  Synchronous; reports the first flat index.
cm_status cm_verify_ex(cm_ctx* c, int32_t scope, int64_t* mismatch, int32_t* what, void* stream) {
    if (!c || !mismatch) return CM_ERR_ARG;
    *mismatch = -1;
    if (what) *what = -1;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->connected || c->no_tap || c->no_shadow) return fail(c, CM_ERR_STATE, "no shadow to verify");
    if (scope <= 0 || scope > (CM_VERIFY_SHADOW | CM_VERIFY_HOST | CM_VERIFY_RING)) return fail(c, CM_ERR_ARG, "bad scope");
    cudaStream_t s = S(stream);
    CU(cudaStreamSynchronize(s));
    CU(cudaDeviceSynchronize());
    if (c->nf_host[0] >= 0) {
        *mismatch = c->nf_host[1];
        if (what) *what = 4;
        return check_nf(c);
    }
    const int64_t T = c->train_step;
    const int64_t step = c->hdr->shadow_step;
    if (step < 0) return fail(c, CM_ERR_STATE, "shadow has no published step");
    unsigned long long init = ~0ull;
    CU(cudaMemcpy(c->d_bad, &init, sizeof init, cudaMemcpyHostToDevice));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((c->shard_numel + 255) / 256, c->misc_blocks));
    if (scope & CM_VERIFY_SHADOW) {
        if (step != T)
            return fail(c, CM_ERR_STATE, "shadow published step %lld, training is at step %lld", (long long)step,
                        (long long)T);
        // the HBM working half, and (HOST placement) the persisted host snapshot if it is at
        // the same step (with persist_every K > 1 it is usually older: CM_VERIFY_HOST)
        const int h = (int)(step & 1);
        int hhalf = -1;
        if (c->shadow_place == CM_SHADOW_HOST)
            for (int i = 0; i < 2; ++i)
                if (c->hdr->half_step[i] == step) hhalf = i;
        for (int which = 0; which < (hhalf >= 0 ? 2 : 1); ++which) {
            const float* src[3];
            for (int a = 0; a < 3; ++a) src[a] = which == 0 ? c->sd[h][a] : to_dev(c, c->sh[hhalf][a]);
            compare_kernel<<<grid, 256, 0, s>>>(src[0], src[1], src[2], c->p, c->m, c->v, c->d_buckets,
                                                (int)c->buckets.size(), c->n, c->rank, 0, c->shard_numel, c->d_bad,
                                                c->zero1 ? 1 : 0);
            c->launches++;
            CHECK_LAUNCH();
        }
    }
    if ((scope & CM_VERIFY_RING) && T >= 1) {
        // the tapped gradients of iteration T-1 (ring slot (T-1) mod D, shard-local, host memory)
        // vs what the training step consumed: shard r of the grad buffer (the caller has not
        // overwritten it since the step), or with ZeRO-1 the staging half it read
        const int slot = (int)((T - 1) % c->D);
        if (c->grads_step != T)
            return fail(c, CM_ERR_STATE, "CM_VERIFY_RING: no training step since the restore (the gradient "
                                         "buffers hold nothing of step %lld)", (long long)T);
        if (!slot_complete(c->seg, c->hdr, c->D, (int)c->buckets.size(), T)) {
            *mismatch = -1;
            if (what) *what = 5;
            return fail(c, CM_ERR_INVARIANT, "ring slot %d does not hold a complete step %lld", slot, (long long)T);
        }
        const void* ref = c->grad;
        int ref_flat = 1;
        if (c->zero1) {
            const int hh = (int)((T - 1) & 1);
            if (c->stage_iter[hh] != T - 1) return fail(c, CM_ERR_STATE, "ZeRO-1 staging half was reused");
            ref = c->stage_buf[hh];
            ref_flat = 0;
        }
        compare_grads_kernel<<<grid, 256, 0, s>>>(ring_slot_dev(c, slot), ref, ref_flat, c->d_buckets,
                                                  (int)c->buckets.size(), c->n, c->rank, c->shard_numel, c->es,
                                                  c->d_bad);
        c->launches++;
        CHECK_LAUNCH();
    }
    if ((scope & CM_VERIFY_HOST) && c->shadow_place == CM_SHADOW_HOST) {
        int64_t gap = -1;
        cm_status st = verify_host_log(c, T, s, &gap);
        if (st != CM_OK) return st;
        if (gap >= 0) {
            if (what) *what = 5;
            return fail(c, CM_ERR_INVARIANT, "the host log cannot reach training step %lld (no snapshot <= it "
                        "rolls forward over complete ring slots; newest usable %lld)", (long long)T, (long long)gap);
        }
    }
    unsigned long long bad = 0;
    CU(cudaMemcpyAsync(&bad, c->d_bad, sizeof bad, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    c->last_s = s;
    c->last_kind = 0;
    if (bad == ~0ull) return CM_OK;
    *mismatch = (int64_t)(bad >> 2);
    const int w = (int)(bad & 3);
    if (what) *what = w;
    static const char* names[4] = {"p", "m", "v", "ring gradient"};
    return fail(c, CM_ERR_INVARIANT, "checkpoint != training at flat index %llu (%s; step %lld, scope %d)",
                bad >> 2, names[w], (long long)T, scope);
}

cm_status cm_verify(cm_ctx* c, int64_t* mismatch, void* stream) {
    return cm_verify_ex(c, CM_VERIFY_SHADOW, mismatch, nullptr, stream);
}

// ---------------------------------------------------------------- restore
// Reading R21.  Shard k holds snapshots in its two
// halves (valid steps) and a ring of tapped gradients.  It can reach step x if some valid
// snapshot b <= x exists and every step b+1..x can be rolled forward: ring slot (s-1) mod D
// has all bucket flags == s and a scalar record tagged s.  hi_k = the largest reachable
// step; I = min_k hi_k; restore fails (UNRECOVERABLE) if some shard cannot reach I.
struct ShardView {
    int64_t half[2];
    std::vector<char> rollable;   // rollable[s - base_lo] for s in (lo, lo + 2D]
    int64_t lo = -1;
};

static bool slot_complete(const char* base, const SegHeader* h, int D, int nb, int64_t s) {
    const SlotMeta* meta = (const SlotMeta*)(base + h->meta_off);
    const volatile uint64_t* flags = (const volatile uint64_t*)(base + h->flags_off);
    const int slot = (int)((s - 1) % D);
    if (h->nf_step >= 0 && s >= h->nf_step) return false;   // never roll forward to a non-finite step
    if (meta[slot].step_tag != s) return false;
    for (int bkt = 0; bkt < nb; ++bkt)
        if (flags[(size_t)slot * nb + bkt] != (uint64_t)s) return false;
    return true;
}

// largest step reachable from snapshot b (b itself if nothing can be rolled forward)
static int64_t roll_limit(const char* base, const SegHeader* h, int D, int nb, int64_t b) {
    int64_t x = b;
    while (x < b + D && slot_complete(base, h, D, nb, x + 1)) ++x;
    return x;
}

struct Reach {
    int64_t snap[2] = {-1, -1};
    int64_t lim[2] = {-1, -1};   // roll_limit from each valid snapshot
    int64_t hi() const { return std::max(lim[0], lim[1]); }
    // best snapshot to reach x from (the newest valid one <= x that rolls to >= x), or -1
    int pick(int64_t x) const {
        int best = -1;
        for (int i = 0; i < 2; ++i)
            if (snap[i] >= 0 && snap[i] <= x && lim[i] >= x && (best < 0 || snap[i] > snap[best])) best = i;
        return best;
    }
};

static Reach reach_of(const SegHeader* h, const char* base, int D, int nb) {
    Reach r;
    for (int i = 0; i < 2; ++i) {
        r.snap[i] = h->half_step[i];
        if (h->nf_step >= 0 && r.snap[i] >= h->nf_step) r.snap[i] = -1;   // conservative: at/after a flagged step
        if (r.snap[i] >= 0) r.lim[i] = roll_limit(base, h, D, nb, r.snap[i]);
    }
    return r;
}

cm_status cm_restore(cm_ctx* c, int64_t* restored, void* stream) {
    if (!c || !restored) return CM_ERR_ARG;
    if (c->cuda_dead) return CM_ERR_CUDA;
    if (!c->connected || c->no_tap || c->no_shadow) return fail(c, CM_ERR_STATE, "no shadow to restore from");
    cudaStream_t s = S(stream);
    CU(cudaDeviceSynchronize());
    // consolidation over all shards (read-only views of the peers' segment headers)
    int64_t I = INT64_MAX;
    std::vector<Reach> R(c->n);
    for (int k = 0; k < c->n; ++k) {
        char name[256];
        snprintf(name, sizeof name, "/%s.r%d", c->shm_name.c_str(), k);
        const char* base = nullptr;
        size_t len = 0;
        if (k == c->rank) {
            base = c->seg;
        } else {
            int fd = shm_open(name, O_RDONLY, 0);
            if (fd < 0) return fail(c, CM_ERR_UNRECOVERABLE, "shadow segment %s missing", name);
            len = c->hdr->ring_off;   // header + meta + flags have the same layout on every rank
            void* mp = mmap(nullptr, len, PROT_READ, MAP_SHARED, fd, 0);
            close(fd);
            if (mp == MAP_FAILED) return fail(c, CM_ERR_UNRECOVERABLE, "mmap %s failed", name);
            base = (const char*)mp;
        }
        const SegHeader* h = (const SegHeader*)base;
        bool ok = h->magic == kMagic && h->layout_hash == c->layout_hash && h->rank == k &&
                  h->ring_depth == c->D;
        if (ok) R[k] = reach_of(h, base, c->D, (int)c->buckets.size());
        if (k != c->rank) munmap((void*)base, len);
        if (!ok) return fail(c, CM_ERR_STATE, "shadow segment %s has a different layout", name);
        if (R[k].hi() < 0) return fail(c, CM_ERR_UNRECOVERABLE, "shard %d has no valid shadow state", k);
        I = std::min(I, R[k].hi());
    }
    for (int k = 0; k < c->n; ++k)
        if (R[k].pick(I) < 0)
            return fail(c, CM_ERR_UNRECOVERABLE, "no common step: shard %d cannot reach step %lld", k, (long long)I);
    // bring this shard to step I: load its snapshot into the HBM half, roll forward
    const Reach& me = R[c->rank];
    const int bi = me.pick(I);
    const int64_t b = me.snap[bi];
    const bool host = c->shadow_place == CM_SHADOW_HOST;
    if (host) {
        for (int a = 0; a < 3; ++a)
            CU(cudaMemcpyAsync(c->sd[b & 1][a], c->sh[bi][a], (size_t)c->shard_numel * 4,
                               cudaMemcpyHostToDevice, s));
        // The roll-forward persists step I over the "older" half.  Never let that be the
        // source snapshot: a kill during the persist would leave this shard only a half
        // beyond I (this shard ran ahead of the consolidation point), and the next restore
        // could not reach I.  A half beyond I is stale anyway (training recomputes it, maybe
        // with other gradients), so it is invalidated first -- by its header step, also when
        // reach_of() ignored it (at or after a non-finite step) -- and becomes the persist
        // target; the source stays intact.  (A half in (b, I] cannot exist: it would roll to
        // I over a subset of the same ring slots, and pick() takes the newest such base.)
        for (int i = 0; i < 2; ++i) {
            if (i != bi && c->hdr->half_step[i] > I) c->hdr->half_step[i] = -1;
            c->hh_step[i] = i == bi ? b : (me.snap[i] > I ? -1 : me.snap[i]);
        }
    } else {
        // DEVICE placement: the HBM halves are the snapshots (half i holds step snap[i], i = step&1)
        for (int i = 0; i < 2; ++i)
            if (c->hdr->half_step[i] > I) c->hdr->half_step[i] = -1;   // training will recompute that step
    }
    for (int64_t st = b + 1; st <= I; ++st) {   // roll forward over the ring
        const int slot = (int)((st - 1) % c->D);
        const SlotMeta* sm = slot_meta(c, slot);
        float f[10];
        for (int k = 0; k < 10; ++k) f[k] = sm->sc[k];
        const StepRec rec = StepRec::from_floats(sm->kind, f);
        cm_status r = shadow_step_enqueue(c, st, rec, s, /*force_persist=*/st == I, nullptr);
        if (r != CM_OK) return r;
    }
    c->hdr->shadow_step = I;
    // shadow shard (HBM half I&1) -> all ranks' p/m/v (NVLink all-gather, one kernel)
    ShardCopyParams P{};
    const int h = (int)(I & 1);
    for (int a = 0; a < 3; ++a) P.src[a] = c->sd[h][a];
    for (int k = 0; k < c->n; ++k) {
        P.dst[0][k] = c->peer_p[k];
        P.dst[1][k] = c->peer_m[k];
        P.dst[2][k] = c->peer_v[k];
    }
    P.buckets = c->d_buckets;
    P.nb = (int)c->buckets.size();
    P.n = c->n;
    P.rank = c->rank;
    P.dir = 1;
    P.barriers = c->barriers ? 1 : 0;
    P.mv_local = c->zero1 ? 1 : 0;
    P.shard_nvec = c->shard_numel / 4;
    P.pads = c->pads;
    P.epoch = ++c->epoch;
    int64_t want = (P.shard_nvec + 255) / 256;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, std::min(c->ar_blocks_max, kMaxBarrierBlocks)));
    shard_copy_kernel<<<grid, 256, 0, s>>>(P);
    c->launches++;
    CHECK_LAUNCH();
    CU(cudaStreamSynchronize(s));
    // Every rank has passed the all-gather's entry barrier, so every rank has computed I from
    // the segment headers: only now may this rank's log change.  Steps beyond I are void
    // (training recomputes them, possibly with different gradients): ring records and tap
    // flags above I are invalidated, so a later restore can never roll forward over a slot
    // that mixes the old run's and the new run's gradients.  The non-finite
    // report is cleared: I precedes it.
    for (int i = 0; i < c->D; ++i) {
        SlotMeta* sm = slot_meta(c, i);
        if (sm->step_tag > I) sm->step_tag = -1;
        volatile uint64_t* fl = slot_flags(c, i);
        for (size_t bk = 0; bk < c->buckets.size(); ++bk)
            if (fl[bk] > (uint64_t)I) fl[bk] = 0;
    }
    c->hdr->nf_index = -1;
    c->hdr->nf_step = -1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    {
        const int64_t none = -1;
        CU(cudaMemcpy(c->d_nf, &none, sizeof none, cudaMemcpyHostToDevice));
    }
    c->last_s = s;
    c->last_kind = 0;
    c->grads_step = -1;   // the gradient buffers hold nothing of step I
    c->cur_iter = I;
    std::fill(c->issued.begin(), c->issued.end(), 0);
    std::fill(c->applied.begin(), c->applied.end(), 0);
    c->applied_count = 0;
    c->issued_count = 0;
    c->train_step = I;
    c->shadow_enq = I;
    c->released_upto = I;   // step I is persisted (HOST) / held in HBM (DEVICE)
    c->stage_iter[0] = c->stage_iter[1] = -1;   // staging halves hold nothing of the new run
    c->dr_b0 = c->dr_b1 = -1;                   // a partial iteration's pending drain is void
    c->dr_bytes = 0;
    c->stage_consumer[0] = c->stage_consumer[1] = false;
    for (int i = 0; i < c->D; ++i) c->slot_sc_step[i] = -1;
    *restored = I;
    return CM_OK;
}

// CM_VERIFY_HOST: rebuild the training step T from the host segment alone -- the newest
// host snapshot b <= T rolled forward over the tapped ring slots b+1..T with their recorded
// scalars, exactly what cm_restore would do -- in chunks of the shadow staging size (scratch
// p/m/v in HBM; the ring is read in place through its device alias), and compare every
// chunk with the training state.  *gap_from >= 0 if no snapshot can reach T.
static cm_status verify_host_log(cm_ctx* c, int64_t T, cudaStream_t s, int64_t* gap_from) {
    *gap_from = -1;
    const int nb = (int)c->buckets.size();
    const Reach me = reach_of(c->hdr, c->seg, c->D, nb);
    const int bi = me.pick(T);
    if (bi < 0) {
        *gap_from = me.hi();
        return CM_OK;
    }
    const int64_t b = me.snap[bi];
    cm_status st = ensure_staging(c);
    if (st != CM_OK) return st;
    const int64_t C = c->stg_elems;
    if (!c->vf_scratch) CU(cudaMalloc(&c->vf_scratch, 3 * (size_t)C * 4));
    float* sp = c->vf_scratch;
    float* smm = sp + C;
    float* sv = smm + C;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((C + 255) / 256, c->misc_blocks));
    std::vector<StepRec> recs;
    for (int64_t x = b + 1; x <= T; ++x) {
        const SlotMeta* m = slot_meta(c, (int)((x - 1) % c->D));
        float f[10];
        for (int k = 0; k < 10; ++k) f[k] = m->sc[k];
        recs.push_back(StepRec::from_floats(m->kind, f));
    }
    for (int64_t lo = 0; lo < c->shard_numel; lo += C) {
        const int64_t len = std::min(C, c->shard_numel - lo);
        CU(cudaMemcpyAsync(sp, c->sh[bi][0] + lo, (size_t)len * 4, cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(smm, c->sh[bi][1] + lo, (size_t)len * 4, cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(sv, c->sh[bi][2] + lo, (size_t)len * 4, cudaMemcpyHostToDevice, s));
        for (int64_t x = b + 1; x <= T; ++x) {
            AdamParams P{};
            P.g = ring_slot_dev(c, (int)((x - 1) % c->D)) + lo * c->es;
            P.n = len;
            set_step(P, recs[x - b - 1]);
            P.p_in = P.p_out = sp;
            P.m_in = P.m_out = smm;
            P.v_in = P.v_out = sv;
            st = launch_adamw(c, P, c->shadow_blocks, s);
            if (st != CM_OK) return st;
        }
        compare_kernel<<<grid, 256, 0, s>>>(sp, smm, sv, c->p, c->m, c->v, c->d_buckets, nb, c->n, c->rank, lo, len,
                                            c->d_bad, c->zero1 ? 1 : 0);
        c->launches++;
        CHECK_LAUNCH();
    }
    return CM_OK;
}

// ---------------------------------------------------------------- introspection
cm_status cm_get_info(const cm_ctx* c, cm_info* o) {
    if (!c || !o) return CM_ERR_ARG;
    memset(o, 0, sizeof *o);
    o->n_buckets = (int32_t)c->buckets.size();
    o->world_size = c->n;
    o->rank = c->rank;
    o->ring_depth = c->D;
    o->grad_dtype = c->dtype;
    o->shadow_place = c->shadow_place;
    o->peers_in_process = c->in_process ? 1 : 0;
    o->drain_ctas = drain_ctas_now(c);
    o->numa_node = c->numa_used;
    o->padded_numel = c->P_pad;
    o->shard_numel = c->shard_numel;
    o->shadow_step = c->hdr ? c->hdr->shadow_step : -1;
    o->launches = c->launches;
    o->layout_hash = c->layout_hash;
    o->nonfinite_step = c->nf_host ? c->nf_host[0] : -1;
    o->nonfinite_index = c->nf_host ? c->nf_host[1] : -1;
    o->persist_every = c->K;
    o->host_half_step[0] = c->hdr ? c->hdr->half_step[0] : -1;
    o->host_half_step[1] = c->hdr ? c->hdr->half_step[1] : -1;
    return CM_OK;
}

cm_status cm_bucket_info(const cm_ctx* c, int32_t b, int64_t* off, int64_t* padded, int64_t* used) {
    if (!c || b < 0 || b >= (int32_t)c->buckets.size()) return CM_ERR_ARG;
    if (off) *off = c->buckets[b].off;
    if (padded) *padded = c->buckets[b].padded;
    if (used) *used = c->buckets[b].used;
    return CM_OK;
}

cm_status cm_shadow_view(const cm_ctx* c, int32_t half, float** p, float** m, float** v) {
    if (!c || half < 0 || half > 1 || !c->hdr) return CM_ERR_ARG;
    float* const* src = c->shadow_place == CM_SHADOW_HOST ? c->sh[half] : c->sd[half];
    if (p) *p = src[0];
    if (m) *m = src[1];
    if (v) *v = src[2];
    return CM_OK;
}

cm_status cm_ring_view(const cm_ctx* c, int32_t slot, void** grads) {
    if (!c || !c->hdr || slot < 0 || slot >= c->D || !grads) return CM_ERR_ARG;
    *grads = c->seg + c->hdr->ring_off + (size_t)slot * c->shard_numel * c->es;
    return CM_OK;
}

cm_status cm_finalize(cm_ctx* c) {
    if (!c) return CM_ERR_ARG;
    if (c->registered || c->pad) cudaSetDevice(c->dev);
    cudaDeviceSynchronize();
    for (auto& e : c->opened) cudaIpcCloseMemHandle(e.second);
    if (c->seg_registered) cudaHostUnregister(c->seg);
    if (c->seg) munmap(c->seg, c->seg_size);
    if (c->shm_fd >= 0) close(c->shm_fd);
    if (c->state_dev_alloc) cudaFree(c->state_dev_alloc);
    if (c->d_buckets) cudaFree(c->d_buckets);
    if (c->pad) cudaFree(c->pad);
    if (c->inbox) cudaFree(c->inbox);
    if (c->nvls) {
        Drv& d = drv();
        d.memUnmap(c->mc_va, c->mc_size);
        d.addrFree(c->mc_va, c->mc_size);
        d.memUnmap(c->uc_va, c->mc_size);
        d.addrFree(c->uc_va, c->mc_size);
        d.mcUnbind(c->mc_handle, (CUdevice)c->dev, 0, c->mc_size);
        d.memRelease(c->mc_phys);
        d.memRelease(c->mc_handle);
    }
    if (c->d_done_ctr) cudaFree(c->d_done_ctr);
    if (c->d_bad) cudaFree(c->d_bad);
    if (c->vf_scratch) cudaFree(c->vf_scratch);
    if (c->ctl) cudaFreeHost(c->ctl);
    if (c->d_nf) cudaFree(c->d_nf);
    for (auto e : c->ev_tap_done) cudaEventDestroy(e);
    for (auto e : c->ev_gstep) if (e) cudaEventDestroy(e);
    for (auto e : c->ev_slot_free) cudaEventDestroy(e);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->cs_tap) cudaStreamDestroy(c->cs_tap);
    for (int i = 0; i < 2; ++i) {
        if (c->stage_buf[i]) cudaFree(c->stage_buf[i]);
        if (c->ev_stage_free[i]) cudaEventDestroy(c->ev_stage_free[i]);
        if (c->ev_ar_done[i]) cudaEventDestroy(c->ev_ar_done[i]);
        if (c->ev_stage_consumed[i]) cudaEventDestroy(c->ev_stage_consumed[i]);
    }
    if (c->ev_ar) cudaEventDestroy(c->ev_ar);
    if (c->stg_ready) {
        for (int j = 0; j < kStages; ++j) {
            cudaFree(c->stg_g[j]);
            cudaEventDestroy(c->ev_stg_free[j]);
            cudaEventDestroy(c->ev_stg_ready[j]);
        }
        cudaEventDestroy(c->ev_fork);
        cudaEventDestroy(c->ev_join);
        cudaStreamDestroy(c->cs_h2d);
        cudaStreamDestroy(c->cs_d2h);
        cudaStreamDestroy(c->cs_k);
    }
    delete c;
    return CM_OK;
}

}  // extern "C"
