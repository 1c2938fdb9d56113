// cm_kernels.cuh -- sm_100a device code of the Checkmate hot path (arXiv 2507.13522).
//
// All kernels are element-local and bandwidth-bound (no tensor cores: nothing on this
// path is a contraction).  Their rooflines and algorithmic bytes are in
// DESIGN.md "Kernels".  Included only by cm_runtime.cu.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace cm {

constexpr int kMaxRanks = 8;
constexpr int kMaxBarrierBlocks = 1024;   // signal-pad slots per region
constexpr int kPadRegions = 2;            // 0 = entry, 1 = exit

// ------------------------------------------------------------------ memory helpers
__device__ __forceinline__ uint4 ld_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// streaming (evict-first) variants for data touched once per launch
__device__ __forceinline__ uint4 ld_cs_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st_cs_v4(void* p, const uint4& v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// NVLink-SHARP multicast store: one 16-byte store through a multicast address, replicated
// by the NVSwitch into every bound device's memory (bits moved as-is, no arithmetic)
__device__ __forceinline__ void mc_st_v4(void* p, const uint4& v) {
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(__uint_as_float(v.x)), "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)),
                    "f"(__uint_as_float(v.w)) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// monotone announce: a barrier slot only ever grows, whatever order two launches' blocks of
// the same index reach it in (atomic max with release semantics, system scope, over NVLink)
__device__ __forceinline__ void max_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("red.release.sys.global.max.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ------------------------------------------------------------------ programmatic dependent launch
// The all-reduce kernels are launched with programmatic stream serialization (PDL): kernel
// N+1 may start as soon as every block of kernel N has passed its entry barrier, so its launch
// and its own entry barrier overlap kernel N's data phase.  Kernel N+1 touches only bucket
// N+1 (disjoint from bucket N everywhere), so it needs no result of kernel N; it waits for
// its predecessor (griddepcontrol.wait) only when that predecessor may have produced its
// gradients (pdl_wait: the previous launch on the stream was not one of our all-reduces).
// Every all-reduce kernel also waits for its predecessor before it EXITS, so kernels still
// complete in stream order: an event or a normal launch after the last bucket's kernel
// sees every earlier bucket's kernel complete, exactly as without PDL.  Both instructions
// are no-ops for a launch without the PDL attribute.
__device__ __forceinline__ void pdl_wait_prior() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_next() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------ cross-GPU barrier
// Pairwise flag exchange between block j of every rank (the grids of one collective
// have equal size on all ranks).  pads[k] is rank k's signal pad (peer-mapped); slot
// (region, block, src) in rank k's pad holds the last epoch src announced to k.
// Epochs increase by one per collective launch and are identical on all ranks (every
// rank issues the same sequence of collectives), so a flag can never be satisfied by a
// stale value; ">=" tolerates a peer that already announced the next epoch.  Announcements
// are an atomic max: with programmatic dependent launch two launches' blocks of one index
// may announce out of order, and a plain store of the older epoch would move the slot
// backwards and strand the peer (measured: a trap under PDL with exit barriers).
struct Pads {
    uint32_t* p[kMaxRanks];
};
__device__ __forceinline__ uint32_t* pad_slot(uint32_t* base, int region, int block, int src) {
    return base + ((size_t)region * kMaxBarrierBlocks + block) * kMaxRanks + src;
}
__device__ __forceinline__ void block_barrier(const Pads& pads, int n, int rank, uint32_t epoch,
                                              int region) {
    __syncthreads();   // all of this block's prior stores are ordered before the release
    if (threadIdx.x < (unsigned)n) {
        const int k = threadIdx.x;
        max_release_sys(pad_slot(pads.p[k], region, blockIdx.x, rank), epoch);
        const uint32_t* mine = pad_slot(pads.p[rank], region, blockIdx.x, k);
        // A peer that never arrives (crashed rank, mismatched call sequence) must not hang
        // the GPU: after ~30 s of waiting the kernel traps and the error surfaces at the
        // next call (CM_ERR_CUDA) instead of a silent deadlock.
        const long long t0 = clock64();
        while ((int)(ld_acquire_sys(mine) - epoch) < 0) {
            __nanosleep(64);
            if (clock64() - t0 > (1ll << 36)) __trap();
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ non-finite detection
// SPEC.md:313, 322 ("non-finite input -> numeric error"); SURVEY 8.b (CM_ERR_INVARIANT) and
// reading R16.  Every kernel that produces a value of the path (the reduced sum, the updated
// p/m/v) checks it; the common case is one untaken branch per vector.  A hit is reported into
// a host-mapped pair nf[0] = step, nf[1] = flat element index (the segment header, so it
// survives the process: restore never rolls forward over a flagged step).  Plain stores, no
// atomics on host memory: an earlier (smaller) step is never overwritten by a later one;
// writers of one step race benignly (any offending index of that step is reported, with a
// flat index from the all-reduce / training kernels preferred over an unknown one, -1).
__device__ __forceinline__ bool nonfinite_f32(float x) { return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u; }
__device__ __forceinline__ bool nonfinite_bf16(uint32_t h) { return (h & 0x7f80u) == 0x7f80u; }
// The report lives twice: h, the host-mapped pair in the segment header (durable, read by
// the host and by restore), and d, a device word holding the step (read by the shadow's
// kernels: thousands of blocks reading one host-mapped word would serialise on PCIe).
struct NfRef {
    volatile int64_t* h;   // [step, index], host-mapped (nullptr: checks off)
    volatile int64_t* d;   // [step], device memory
};
__device__ __noinline__ void nf_report(NfRef nf, int64_t step, int64_t index) {
    const int64_t dc = nf.d[0];
    if (dc < 0 || dc > step) nf.d[0] = step;
    const int64_t cur = nf.h[0];
    if (index < 0) {             // (the shadow: no flat index) never touches the index word
        if (cur < 0 || cur > step) {
            nf.h[0] = step;
            __threadfence_system();
        }
        return;
    }
    if (cur >= 0 && (cur < step || (cur == step && nf.h[1] >= 0))) return;
    nf.h[1] = index;
    __threadfence_system();
    nf.h[0] = step;
    __threadfence_system();
}
// updated state of 4 consecutive elements (index idx0..idx0+3; -1: unknown)
__device__ __forceinline__ void nf_check4(NfRef nf, int64_t step, int64_t idx0, const float4& p,
                                          const float4& m, const float4& v) {
    if (!nf.h) return;
    const float a[4] = {p.x, p.y, p.z, p.w}, b[4] = {m.x, m.y, m.z, m.w}, c[4] = {v.x, v.y, v.z, v.w};
    bool any = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) any |= nonfinite_f32(a[k]) | nonfinite_f32(b[k]) | nonfinite_f32(c[k]);
    if (!any) return;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (nonfinite_f32(a[k]) | nonfinite_f32(b[k]) | nonfinite_f32(c[k])) {
            nf_report(nf, step, idx0 < 0 ? -1 : idx0 + k);
            return;
        }
}
// a stream-ordered kernel of a step that must not run once the step (or an earlier one) was
// flagged: the shadow never applies or publishes a non-finite iteration
__device__ __forceinline__ bool nf_blocked(const volatile int64_t* skip, int64_t step) {
    if (!skip) return false;
    const int64_t s = skip[0];
    return s >= 0 && s <= step;
}

// ------------------------------------------------------------------ dtype traits
// A 16-byte vector of gradients: 4 fp32 or 8 bf16.
struct F32Tag {};
struct BF16Tag {};
template <typename G> struct GT;
template <> struct GT<F32Tag> {
    static constexpr int kPerVec = 4;
    static constexpr int kBytes = 4;
};
template <> struct GT<BF16Tag> {
    static constexpr int kPerVec = 8;
    static constexpr int kBytes = 2;
};

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
// round-to-nearest-even fp32 -> bf16 (reading R25; finite inputs)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t a = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
    uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
    return a | (b << 16);
}

// ------------------------------------------------------------------ counter-based inputs
// SplitMix64 finaliser; h = sm(K ^ i), K = sm(seed ^ r<<48 ^ t)
// computed on the host.  fp32: mant int24, value = mant * 2^(-23-e-s); bf16: mant int8,
// value = mant * 2^(-7-e-s); e = (h>>32)&7.  Exact in the target dtype.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ float pow2i(int k) {   // 2^k for k in the normal range
    return __uint_as_float((uint32_t)(127 + k) << 23);
}
__device__ __forceinline__ float gen_f32(uint64_t K, uint64_t i, int s) {
    uint64_t h = splitmix64(K ^ i);
    int e = (int)((h >> 32) & 7u);
    int mant = (int)(h >> 40) - (1 << 23);
    return __fmul_rn((float)mant, pow2i(-23 - e - s));
}
__device__ __forceinline__ uint32_t gen_bf16bits(uint64_t K, uint64_t i, int s) {
    uint64_t h = splitmix64(K ^ i);
    int e = (int)((h >> 32) & 7u);
    int mant = (int)(h >> 56) - 128;
    return __float_as_uint(__fmul_rn((float)mant, pow2i(-7 - e - s))) >> 16;
}

struct BucketDev {
    int64_t off;      // flat element offset
    int64_t padded;   // E_b
    int64_t used;     // real elements (rest is zero padding)
    int64_t shard_off;// shard-local element offset = off / n
};

// Grid-stride over 16-byte vectors of the flat buffer; a running bucket index locates
// padding (buckets are whole vectors, so a vector never straddles two buckets).
template <typename G>
__global__ void __launch_bounds__(256) gen_grads_kernel(void* __restrict__ out, int64_t nvec,
                                                        const BucketDev* __restrict__ buckets,
                                                        int nb, uint64_t K, int s) {
    constexpr int V = GT<G>::kPerVec;
    int b = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nvec;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = q * V;
        while (b + 1 < nb && i0 >= buckets[b + 1].off) ++b;
        const int64_t lim = buckets[b].off + buckets[b].used;
        uint32_t w[4];
        if constexpr (V == 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                w[k] = (i0 + k < lim) ? __float_as_uint(gen_f32(K, (uint64_t)(i0 + k), s)) : 0u;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t lo = (i0 + 2 * k < lim) ? gen_bf16bits(K, (uint64_t)(i0 + 2 * k), s) : 0u;
                uint32_t hi = (i0 + 2 * k + 1 < lim) ? gen_bf16bits(K, (uint64_t)(i0 + 2 * k + 1), s) : 0u;
                w[k] = lo | (hi << 16);
            }
        }
        st_v4((char*)out + q * 16, make_uint4(w[0], w[1], w[2], w[3]));
    }
}

// p = p_0 (generator, rank 0xFFFF, t 0, s 0, times 2^-5), m = v = 0.
__global__ void __launch_bounds__(256) init_state_kernel(float* __restrict__ p, float* __restrict__ m,
                                                         float* __restrict__ v, int64_t nvec,
                                                         const BucketDev* __restrict__ buckets, int nb,
                                                         uint64_t K) {
    int b = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nvec;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = q * 4;
        while (b + 1 < nb && i0 >= buckets[b + 1].off) ++b;
        const int64_t lim = buckets[b].off + buckets[b].used;
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            w[k] = (i0 + k < lim) ? __float_as_uint(__fmul_rn(gen_f32(K, (uint64_t)(i0 + k), 0), 0.03125f)) : 0u;
        st_v4(p + i0, make_uint4(w[0], w[1], w[2], w[3]));
        if (m) {   // (ZeRO-1: m, v are shard-local and zeroed separately)
            st_v4(m + i0, make_uint4(0, 0, 0, 0));
            st_v4(v + i0, make_uint4(0, 0, 0, 0));
        }
    }
}

// ------------------------------------------------------------------ RS + tap + AG
// One launch per (bucket, iteration) per rank.  Rank r reduces shard r of the bucket:
// for every 16-byte vector of the shard, read it from all n ranks' grad buffers (n-1 of
// them over NVLink), sum in rank order in fp32 registers (seeded with rank 0's value,
// readings R2/R3), round once to bf16 for bf16 grads (R14), then store the same
// registers to (a) the host ring (the tap, exactly once box-wide) and (b) shard r of all
// n ranks' grad buffers (the all-gather).  In place is race-free: rank r is the only
// rank that reads or writes shard r of any buffer, and a thread writes an element only
// after it has read that element from all n ranks.
struct ArParams {
    char* buf[kMaxRanks];   // grad buffer of rank k + bucket byte offset + shard byte offset
    char* tap;              // host-mapped ring slot + shard byte offset (nullptr: no tap)
    int64_t nvec;           // 16-byte vectors in the shard
    Pads pads;
    uint32_t epoch;
    int rank;
    int barriers;           // 0 when all ranks live in this process (virtual ranks)
    int exit_barrier;       // 0: the iteration's fence is the training step's entry barrier
    int ag;                 // 0 when n == 1 (the reduced value equals the local value)
    unsigned long long* done_ctr;  // device counter: last block to finish publishes the flag
    unsigned long long done_target;
    volatile uint64_t* tap_flag;   // host-mapped (slot, bucket, rank) flag; nullptr: none
    uint64_t tap_flag_value;       // iteration + 1
    NfRef nf;                      // non-finite report (nf.h = nullptr: off)
    int64_t elem0;                 // flat element index of the shard's first element
    int64_t nf_step;               // the step that applies this reduce (iteration + 1)
    int pdl_wait;                  // 1: wait for the predecessor kernel (it may have written
                                   // this bucket's gradients) before the entry barrier
    int pdl_mode;                  // experiments: bit 0 = no wait for the predecessor at exit,
                                   // bit 1 = trigger the dependents after the data phase
    int tma_tile;                  // bulk-copy pipeline: bytes per rank per stage (multiple of 128)
};

// a reduced 16-byte vector (the value the tap and the all-gather store) is finite?  Else
// report the first non-finite element (flat index elem0 + q*V + k).
template <typename G>
__device__ __forceinline__ void nf_check_vec(NfRef nf, int64_t step, int64_t elem0, const uint4& r) {
    if (!nf.h) return;
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
    if constexpr (std::is_same<G, F32Tag>::value) {
        bool any = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) any |= nonfinite_f32(__uint_as_float(w[k]));
        if (!any) return;
        for (int k = 0; k < 4; ++k)
            if (nonfinite_f32(__uint_as_float(w[k]))) { nf_report(nf, step, elem0 + k); return; }
    } else {
        bool any = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) any |= nonfinite_bf16(w[k] & 0xFFFFu) | nonfinite_bf16(w[k] >> 16);
        if (!any) return;
        for (int k = 0; k < 8; ++k)
            if (nonfinite_bf16((w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu)) { nf_report(nf, step, elem0 + k); return; }
    }
}

template <typename G, int N>
__device__ __forceinline__ uint4 reduce_vec(const uint4 (&x)[N]) {
    if constexpr (std::is_same<G, F32Tag>::value) {
        float a0 = __uint_as_float(x[0].x), a1 = __uint_as_float(x[0].y);
        float a2 = __uint_as_float(x[0].z), a3 = __uint_as_float(x[0].w);
#pragma unroll
        for (int k = 1; k < N; ++k) {
            a0 = __fadd_rn(a0, __uint_as_float(x[k].x));
            a1 = __fadd_rn(a1, __uint_as_float(x[k].y));
            a2 = __fadd_rn(a2, __uint_as_float(x[k].z));
            a3 = __fadd_rn(a3, __uint_as_float(x[k].w));
        }
        return make_uint4(__float_as_uint(a0), __float_as_uint(a1), __float_as_uint(a2),
                          __float_as_uint(a3));
    } else {
        if constexpr (N == 1) return x[0];   // RNE(upcast(b)) == b
        float a[8];
        a[0] = bf16lo(x[0].x); a[1] = bf16hi(x[0].x); a[2] = bf16lo(x[0].y); a[3] = bf16hi(x[0].y);
        a[4] = bf16lo(x[0].z); a[5] = bf16hi(x[0].z); a[6] = bf16lo(x[0].w); a[7] = bf16hi(x[0].w);
#pragma unroll
        for (int k = 1; k < N; ++k) {
            a[0] = __fadd_rn(a[0], bf16lo(x[k].x)); a[1] = __fadd_rn(a[1], bf16hi(x[k].x));
            a[2] = __fadd_rn(a[2], bf16lo(x[k].y)); a[3] = __fadd_rn(a[3], bf16hi(x[k].y));
            a[4] = __fadd_rn(a[4], bf16lo(x[k].z)); a[5] = __fadd_rn(a[5], bf16hi(x[k].z));
            a[6] = __fadd_rn(a[6], bf16lo(x[k].w)); a[7] = __fadd_rn(a[7], bf16hi(x[k].w));
        }
        return make_uint4(pack_bf16x2(a[0], a[1]), pack_bf16x2(a[2], a[3]), pack_bf16x2(a[4], a[5]),
                          pack_bf16x2(a[6], a[7]));
    }
}

constexpr int kArThreads = 512;
constexpr int kArUnroll = 2;

template <typename G, int N>
__device__ __forceinline__ void ar_load(const ArParams& P, int64_t q, uint4 (&x)[N]) {
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = ld_v4(P.buf[k] + q * 16);
}
template <typename G, int N>
__device__ __forceinline__ void ar_reduce_store(const ArParams& P, int64_t q, const uint4 (&x)[N]) {
    const uint4 r = reduce_vec<G, N>(x);
    const int64_t off = q * 16;
    nf_check_vec<G>(P.nf, P.nf_step, P.elem0 + q * GT<G>::kPerVec, r);
    if (P.tap) st_cs_v4(P.tap + off, r);
    if (P.ag) {
#pragma unroll
        for (int k = 0; k < N; ++k) st_v4(P.buf[k] + off, r);
    }
}
// tap flag of the direct tap (last block publishes) and the optional exit barrier
template <int N>
__device__ __forceinline__ void ar_epilogue(const ArParams& P) {
    if (P.tap_flag) {
        // every tap store of this block is visible system-wide before the block is
        // counted; the last block publishes the (slot, bucket, rank) flag for restore
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long prev = atomicAdd(P.done_ctr, 1ull);
            if (prev + 1 == P.done_target) {
                __threadfence_system();
                *P.tap_flag = P.tap_flag_value;
            }
        }
    }
    // bucket complete everywhere; skipped when the training step's entry barrier fences the
    // whole iteration instead (the next bucket's kernel then overlaps this one's store tail)
    if (P.barriers && P.exit_barrier) block_barrier(P.pads, N, P.rank, P.epoch, 1);
}

template <typename G, int N>
__global__ void __launch_bounds__(kArThreads) rs_tap_ag_kernel(const ArParams P) {
    if (P.pdl_wait) pdl_wait_prior();
    if (P.barriers) block_barrier(P.pads, N, P.rank, P.epoch, 0);   // peers' grads are ready
    if (!(P.pdl_mode & 2)) pdl_launch_next();                       // the next bucket may launch

    const int64_t stride = (int64_t)gridDim.x * kArThreads;
    int64_t q = blockIdx.x * (int64_t)kArThreads + threadIdx.x;
    for (; q + (kArUnroll - 1) * stride < P.nvec; q += kArUnroll * stride) {
        uint4 x[kArUnroll][N];
#pragma unroll
        for (int u = 0; u < kArUnroll; ++u) ar_load<G, N>(P, q + u * stride, x[u]);
#pragma unroll
        for (int u = 0; u < kArUnroll; ++u) ar_reduce_store<G, N>(P, q + u * stride, x[u]);
    }
    for (; q < P.nvec; q += stride) {
        uint4 x[N];
        ar_load<G, N>(P, q, x);
        ar_reduce_store<G, N>(P, q, x);
    }
    if (P.pdl_mode & 2) pdl_launch_next();
    ar_epilogue<N>(P);
    if (!(P.pdl_mode & 1)) pdl_wait_prior();   // complete after the predecessor (stream-order completion)
}

// Software-pipelined variant (cm_set_param("ar_impl", 1)): one block per SM, each thread
// walks its vectors with the n loads of vector q + stride in flight while vector q is
// reduced and stored, so the inbound (reads) and outbound (all-gather stores) directions
// of the links are busy at the same time instead of in alternating phases.
template <typename G, int N>
__global__ void __launch_bounds__(kArThreads, 1) rs_tap_ag_pipe_kernel(const ArParams P) {
    if (P.pdl_wait) pdl_wait_prior();
    if (P.barriers) block_barrier(P.pads, N, P.rank, P.epoch, 0);   // peers' grads are ready
    pdl_launch_next();
    const int64_t stride = (int64_t)gridDim.x * kArThreads;
    int64_t q = blockIdx.x * (int64_t)kArThreads + threadIdx.x;
    if (q < P.nvec) {
        uint4 cur[N];
        ar_load<G, N>(P, q, cur);
        for (; q < P.nvec; q += stride) {
            uint4 nxt[N];
            const int64_t qn = q + stride;
            if (qn < P.nvec) ar_load<G, N>(P, qn, nxt);
            ar_reduce_store<G, N>(P, q, cur);
#pragma unroll
            for (int k = 0; k < N; ++k) cur[k] = nxt[k];
        }
    }
    ar_epilogue<N>(P);
    pdl_wait_prior();
}

// ------------------------------------------------------------------ one-shot push AR
// small buckets (Llama's 16 KiB norm pairs) are latency-bound, and the
// two-shot kernel pays a pull round trip over NVLink plus an exit barrier for the remote
// all-gather stores.  One-shot push: every rank stores its whole bucket into slot [rank] of
// every peer's inbox (posted NVLink writes), one pairwise block barrier, then every rank
// sums all n copies in rank order from its LOCAL inbox (identical R on every rank: same
// operands, same order) and writes its own grad buffer only.  Rank r taps only the
// elements of its own shard, so the tap stays exactly once box-wide.  Traffic per GPU is
// (n-1) S_b each way instead of 2(n-1)/n S_b: only worth it where latency dominates.
// Inbox halves alternate with the launch epoch; between two launches that use the same
// half every rank has passed a barrier of the launch in between, so a slot is never
// overwritten while its owner still reads it.
struct OsParams {
    char* own;                     // this rank's grad buffer + bucket byte offset
    char* push[kMaxRanks];         // peer k's inbox slot [rank] (unused for k == rank)
    const char* inbox[kMaxRanks];  // this rank's inbox slot [k] (unused for k == rank)
    char* tap;                     // tap target of this rank's shard (nullptr: no tap)
    char* mc;                      // NVLS: multicast address of slot [rank] (nullptr: unicast)
    int64_t nvec;                  // 16-byte vectors in the bucket
    int64_t shard_lo, shard_hi;    // this rank's shard, in vectors
    int64_t shard_vec;             // vectors per shard (E_b / n * sizeof(G) / 16)
    int rs_only;                   // ZeRO-1: push shard k to rank k only, reduce the own shard
                                   // into the tap target, leave the grad buffer untouched
    Pads pads;
    uint32_t epoch;
    int rank;
    unsigned long long* done_ctr;
    unsigned long long done_target;
    volatile uint64_t* tap_flag;
    uint64_t tap_flag_value;
    NfRef nf;                      // non-finite report (see ArParams)
    int64_t elem0;                 // flat element index of the bucket's first element
    int64_t nf_step;
};

constexpr int kOsThreads = 256;

template <typename G, int N>
__global__ void __launch_bounds__(kOsThreads) os_tap_kernel(const OsParams P) {
    const int64_t stride = (int64_t)gridDim.x * kOsThreads;
    const int64_t q0 = blockIdx.x * (int64_t)kOsThreads + threadIdx.x;
    if (P.rs_only) {                                         // push shard k to its owner only
        for (int64_t q = q0; q < P.nvec; q += stride) {
            const int k = (int)(q / P.shard_vec);
            if (k != P.rank) st_v4(P.push[k] + q * 16, ld_v4(P.own + q * 16));
        }
    } else if (P.mc) {                                       // push once: the switch replicates
        for (int64_t q = q0; q < P.nvec; q += stride) mc_st_v4(P.mc + q * 16, ld_v4(P.own + q * 16));
        __threadfence_system();
    } else {                                                 // push n-1 unicast copies
        for (int64_t q = q0; q < P.nvec; q += stride) {
            const uint4 x = ld_v4(P.own + q * 16);
#pragma unroll
            for (int k = 0; k < N; ++k)
                if (k != P.rank) st_v4(P.push[k] + q * 16, x);
        }
    }
    block_barrier(P.pads, N, P.rank, P.epoch, 0);            // every rank's chunk arrived
    for (int64_t q = q0; q < P.nvec; q += stride) {          // reduce from the local inbox
        if (P.rs_only && (q < P.shard_lo || q >= P.shard_hi)) continue;
        uint4 x[N];
#pragma unroll
        for (int k = 0; k < N; ++k) x[k] = ld_v4((k == P.rank ? (const char*)P.own : P.inbox[k]) + q * 16);
        const uint4 r = reduce_vec<G, N>(x);
        nf_check_vec<G>(P.nf, P.nf_step, P.elem0 + q * GT<G>::kPerVec, r);
        if (!P.rs_only) st_v4(P.own + q * 16, r);
        if (P.tap && q >= P.shard_lo && q < P.shard_hi) st_cs_v4(P.tap + (q - P.shard_lo) * 16, r);
    }
    if (P.tap_flag) {
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long prev = atomicAdd(P.done_ctr, 1ull);
            if (prev + 1 == P.done_target) {
                __threadfence_system();
                *P.tap_flag = P.tap_flag_value;
            }
        }
    }
}

// ------------------------------------------------------------------ AdamW
// Canonical fp32 op sequence (reading R4), each op IEEE round-to-nearest, no FMA:
//   g = R*inv_n; m = B1*m + c1*g; v = B2*v + c2*(g*g); mh = m/bc1; vh = v/bc2;
//   d = sqrt(vh) + eps; p = p - lr*(mh/d + wd*p)
struct AdamScalars {
    float c1, c2, B1, B2, bc1, bc2, inv_n, lr, eps, wd;
};

// IEEE-exact x / y and sqrt(x) that keep a zero operand off the slow path: the compiled
// __fdiv_rn / __fsqrt_rn check their operands (FCHK) and branch to a subroutine for zero
// and denormal inputs, and one such lane stalls its whole warp.  Zero moments are common
// (an element whose gradient has been exactly zero since the start: untouched embedding
// rows, 1 in 256 bf16 generator values), so the zero case is answered directly:
// +-0 / y = +-0 for y > 0 and sqrt(+-0) = +-0, both exactly what IEEE 754 returns.
__device__ __forceinline__ float div_rn_z(float x, float y) {
    const bool z = (x == 0.0f) && (y > 0.0f);
    const float q = __fdiv_rn(z ? 1.0f : x, z ? 1.0f : y);
    return z ? x : q;
}
__device__ __forceinline__ float sqrt_rn_z(float x) {
    const bool z = (x == 0.0f);
    const float r = __fsqrt_rn(z ? 1.0f : x);
    return z ? x : r;
}

__device__ __forceinline__ void adamw_elem(float R, const AdamScalars& s, float& p, float& m, float& v) {
    const float g = __fmul_rn(R, s.inv_n);
    const float mm = __fadd_rn(__fmul_rn(s.B1, m), __fmul_rn(s.c1, g));
    const float vv = __fadd_rn(__fmul_rn(s.B2, v), __fmul_rn(s.c2, __fmul_rn(g, g)));
    const float mh = div_rn_z(mm, s.bc1);
    const float vh = div_rn_z(vv, s.bc2);
    const float d = __fadd_rn(sqrt_rn_z(vh), s.eps);
    const float upd = __fadd_rn(div_rn_z(mh, d), __fmul_rn(s.wd, p));
    p = __fsub_rn(p, __fmul_rn(s.lr, upd));
    m = mm;
    v = vv;
}

// SGD with momentum (reading R27), fp32, no FMA:
//   g = R*inv_n; d = g (wd_on = 0) or g + wd*p (wd_on = 1); buf = mu*buf + d; p = p - lr*buf
// The velocity lives in the m array; v is not touched.
struct SgdScalars {
    float mu, inv_n, lr, wd;
    int wd_on;
};

__device__ __forceinline__ void sgd_elem(float R, const SgdScalars& q, float& p, float& buf) {
    const float g = __fmul_rn(R, q.inv_n);
    const float d = q.wd_on ? __fadd_rn(g, __fmul_rn(q.wd, p)) : g;
    const float b = __fadd_rn(__fmul_rn(q.mu, buf), d);
    p = __fsub_rn(p, __fmul_rn(q.lr, b));
    buf = b;
}

// Optimizer selector of the element-local step kernels (same data path, different op).
enum OptKind : int { kOptAdamW = 0, kOptSgd = 1 };

// A work item = 8 consecutive elements (two float4 of state; 32 B of fp32 grads or 16 B
// of bf16 grads).  All arrays are 16-byte aligned and a multiple of 8 elements long
// except possibly a 4-element tail for fp32 (handled by the tail item path).
// In/out arrays may alias (training: in place) or not (shadow: ping-pong halves).
struct AdamParams {
    const void* g;
    const float* p_in; const float* m_in; const float* v_in;
    float* p_out; float* m_out; float* v_out;
    int64_t n;          // elements (multiple of 4)
    AdamScalars s;
    SgdScalars q;       // used by the kOptSgd instances (v_in / v_out unused there)
    volatile float* hp_rec;        // host-mapped ring-slot scalar record (or nullptr)
    volatile int32_t* hp_kind;     // host-mapped record: optimizer kind
    volatile int64_t* hp_tag;      // written after the record: the step
    float rec[10];                 // the record's scalars (AdamScalars or SgdScalars)
    int32_t rec_kind;
    int64_t step;
    // iteration fence (training step only, multi-process, lazy all-reduce exits): block j
    // waits for block j of every rank, i.e. for every rank to have finished ALL its
    // all-reduce kernels of the iteration -- their all-gather stores into this rank's grad
    // buffer have landed, and nobody still reads this rank's grads when the next backward
    // overwrites them
    Pads pads;
    uint32_t epoch;
    int fence_n, fence_rank;       // fence_n = 0: no fence
    NfRef nf;                      // non-finite report of the updated state (nf.h = nullptr: off)
    int64_t nf_base;               // flat index of element 0 of this launch (-1: not flat, e.g. shadow)
    const volatile int64_t* skip_nf;  // shadow: do nothing if the step (or an earlier) was flagged
                                      // (the device word NfRef::d)
};

// whole-block early exit of a shadow kernel whose step was flagged non-finite (one host read
// per block)
template <typename PT>
__device__ __forceinline__ bool block_nf_blocked(const PT& P) {
    if (!P.skip_nf) return false;
    __shared__ int blk;
    if (threadIdx.x == 0) blk = nf_blocked(P.skip_nf, P.step) ? 1 : 0;
    __syncthreads();
    return blk != 0;
}
__device__ __forceinline__ int64_t nf_idx(int64_t base, int64_t e) { return base < 0 ? -1 : base + e; }

// the step's scalars into the host-mapped ring-slot record, then its tag (one thread)
template <typename PT>
__device__ __forceinline__ void write_record(const PT& P) {
    if (!P.hp_rec) return;
    for (int k = 0; k < 10; ++k) P.hp_rec[k] = P.rec[k];
    *P.hp_kind = P.rec_kind;
    __threadfence_system();
    *P.hp_tag = P.step;
}

constexpr int kAdamThreads = 256;

template <typename G>
__device__ __forceinline__ void adamw_item(const AdamParams& P, int64_t e) {
    // e: first element of the 8-element item (e + 8 <= n).  __ldcs/__stcs: evict-first
    // streaming accesses (every byte is touched once per launch).
    float4 g0, g1;
    if constexpr (std::is_same<G, F32Tag>::value) {
        g0 = __ldcs(reinterpret_cast<const float4*>((const float*)P.g + e));
        g1 = __ldcs(reinterpret_cast<const float4*>((const float*)P.g + e + 4));
    } else {
        const uint4 gb = __ldcs(reinterpret_cast<const uint4*>((const uint16_t*)P.g + e));
        g0 = make_float4(bf16lo(gb.x), bf16hi(gb.x), bf16lo(gb.y), bf16hi(gb.y));
        g1 = make_float4(bf16lo(gb.z), bf16hi(gb.z), bf16lo(gb.w), bf16hi(gb.w));
    }
    float4 p0 = __ldcs(reinterpret_cast<const float4*>(P.p_in + e));
    float4 p1 = __ldcs(reinterpret_cast<const float4*>(P.p_in + e + 4));
    float4 m0 = __ldcs(reinterpret_cast<const float4*>(P.m_in + e));
    float4 m1 = __ldcs(reinterpret_cast<const float4*>(P.m_in + e + 4));
    float4 v0 = __ldcs(reinterpret_cast<const float4*>(P.v_in + e));
    float4 v1 = __ldcs(reinterpret_cast<const float4*>(P.v_in + e + 4));
    adamw_elem(g0.x, P.s, p0.x, m0.x, v0.x); adamw_elem(g0.y, P.s, p0.y, m0.y, v0.y);
    adamw_elem(g0.z, P.s, p0.z, m0.z, v0.z); adamw_elem(g0.w, P.s, p0.w, m0.w, v0.w);
    adamw_elem(g1.x, P.s, p1.x, m1.x, v1.x); adamw_elem(g1.y, P.s, p1.y, m1.y, v1.y);
    adamw_elem(g1.z, P.s, p1.z, m1.z, v1.z); adamw_elem(g1.w, P.s, p1.w, m1.w, v1.w);
    nf_check4(P.nf, P.step, nf_idx(P.nf_base, e), p0, m0, v0);
    nf_check4(P.nf, P.step, nf_idx(P.nf_base, e + 4), p1, m1, v1);
    __stcs(reinterpret_cast<float4*>(P.p_out + e), p0);
    __stcs(reinterpret_cast<float4*>(P.p_out + e + 4), p1);
    __stcs(reinterpret_cast<float4*>(P.m_out + e), m0);
    __stcs(reinterpret_cast<float4*>(P.m_out + e + 4), m1);
    __stcs(reinterpret_cast<float4*>(P.v_out + e), v0);
    __stcs(reinterpret_cast<float4*>(P.v_out + e + 4), v1);
}

template <typename G>
__global__ void __launch_bounds__(kAdamThreads) adamw_kernel(const AdamParams P) {
    if (block_nf_blocked(P)) return;
    const int64_t items = P.n / 8;
    const int64_t stride = (int64_t)gridDim.x * kAdamThreads;
    int64_t q = blockIdx.x * (int64_t)kAdamThreads + threadIdx.x;
    for (; q + stride < items; q += 2 * stride) {
        adamw_item<G>(P, q * 8);
        adamw_item<G>(P, (q + stride) * 8);
    }
    for (; q < items; q += stride) adamw_item<G>(P, q * 8);
    // fp32 tail of 4 elements (n % 8 == 4)
    if (blockIdx.x == 0 && threadIdx.x == 0 && (P.n & 7)) {
        for (int64_t e = items * 8; e < P.n; ++e) {
            float R;
            if constexpr (std::is_same<G, F32Tag>::value) R = ((const float*)P.g)[e];
            else R = __uint_as_float(((uint32_t)((const uint16_t*)P.g)[e]) << 16);
            float p = P.p_in[e], m = P.m_in[e], v = P.v_in[e];
            adamw_elem(R, P.s, p, m, v);
            nf_check4(P.nf, P.step, nf_idx(P.nf_base, e), make_float4(p, 0.f, 0.f, 0.f), make_float4(m, 0.f, 0.f, 0.f),
                      make_float4(v, 0.f, 0.f, 0.f));
            P.p_out[e] = p; P.m_out[e] = m; P.v_out[e] = v;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) write_record(P);
}

// ------------------------------------------------------------------ AdamW, warp-tiled
// Same arithmetic; each warp owns 256-element tiles and every warp-wide 16-byte access is
// one contiguous 512-byte run (lane l: elements 4l..4l+3 and 128+4l..128+4l+3), so each
// load instruction touches exactly 4 full 128-byte lines.  Two tiles are loaded before
// either is stored (16 independent 16-byte loads in flight per thread).
constexpr int kWarpTile = 256;

template <typename G, int OPT = kOptAdamW>
__device__ __forceinline__ void wt_load(const AdamParams& P, int64_t e, float4& g, float4& p, float4& m, float4& v) {
    if constexpr (std::is_same<G, F32Tag>::value) {
        g = __ldcs(reinterpret_cast<const float4*>((const float*)P.g + e));
    } else {
        const uint2 w = __ldcs(reinterpret_cast<const uint2*>((const uint16_t*)P.g + e));
        g = make_float4(bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y));
    }
    p = __ldcs(reinterpret_cast<const float4*>(P.p_in + e));
    m = __ldcs(reinterpret_cast<const float4*>(P.m_in + e));
    if constexpr (OPT == kOptAdamW) v = __ldcs(reinterpret_cast<const float4*>(P.v_in + e));
}
template <int OPT = kOptAdamW>
__device__ __forceinline__ void wt_compute_store(const AdamParams& P, int64_t e, const float4& g, float4 p,
                                                 float4 m, float4 v) {
    if constexpr (OPT == kOptAdamW) {
        adamw_elem(g.x, P.s, p.x, m.x, v.x);
        adamw_elem(g.y, P.s, p.y, m.y, v.y);
        adamw_elem(g.z, P.s, p.z, m.z, v.z);
        adamw_elem(g.w, P.s, p.w, m.w, v.w);
    } else {
        sgd_elem(g.x, P.q, p.x, m.x);
        sgd_elem(g.y, P.q, p.y, m.y);
        sgd_elem(g.z, P.q, p.z, m.z);
        sgd_elem(g.w, P.q, p.w, m.w);
    }
    nf_check4(P.nf, P.step, nf_idx(P.nf_base, e), p, m, v);
    __stcs(reinterpret_cast<float4*>(P.p_out + e), p);
    __stcs(reinterpret_cast<float4*>(P.m_out + e), m);
    if constexpr (OPT == kOptAdamW) __stcs(reinterpret_cast<float4*>(P.v_out + e), v);
}

// PAIR: two tiles per iteration (16 loads in flight per thread, ~100 registers, 2 blocks of
// 256 per SM); !PAIR: one tile per iteration (8 loads, <= 64 registers, 4 blocks per SM:
// twice the warps to overlap one warp's IEEE div/sqrt chain with other warps' loads)
template <typename G, int OPT, bool PAIR = true>
__device__ __forceinline__ void wt_body(const AdamParams& P) {
    if (block_nf_blocked(P)) return;
    if (P.fence_n) block_barrier(P.pads, P.fence_n, P.fence_rank, P.epoch, 0);
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)kAdamThreads + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kAdamThreads) >> 5;
    const int64_t tiles = P.n / kWarpTile;
    int64_t t = warp;
    for (; PAIR && t + nwarps < tiles; t += 2 * nwarps) {
        const int64_t a0 = t * kWarpTile + 4 * lane, a1 = a0 + 128;
        const int64_t b0 = (t + nwarps) * kWarpTile + 4 * lane, b1 = b0 + 128;
        float4 g[4], p[4], m[4], v[4] = {};
        wt_load<G, OPT>(P, a0, g[0], p[0], m[0], v[0]);
        wt_load<G, OPT>(P, a1, g[1], p[1], m[1], v[1]);
        wt_load<G, OPT>(P, b0, g[2], p[2], m[2], v[2]);
        wt_load<G, OPT>(P, b1, g[3], p[3], m[3], v[3]);
        wt_compute_store<OPT>(P, a0, g[0], p[0], m[0], v[0]);
        wt_compute_store<OPT>(P, a1, g[1], p[1], m[1], v[1]);
        wt_compute_store<OPT>(P, b0, g[2], p[2], m[2], v[2]);
        wt_compute_store<OPT>(P, b1, g[3], p[3], m[3], v[3]);
    }
    for (; t < tiles; t += nwarps) {
        const int64_t a0 = t * kWarpTile + 4 * lane, a1 = a0 + 128;
        float4 g[2], p[2], m[2], v[2] = {};
        wt_load<G, OPT>(P, a0, g[0], p[0], m[0], v[0]);
        wt_load<G, OPT>(P, a1, g[1], p[1], m[1], v[1]);
        wt_compute_store<OPT>(P, a0, g[0], p[0], m[0], v[0]);
        wt_compute_store<OPT>(P, a1, g[1], p[1], m[1], v[1]);
    }
    // tail: n % 256 elements (a multiple of 4), one float4 group per thread of block 0
    if (blockIdx.x == 0) {
        const int64_t e = tiles * kWarpTile + 4 * (int64_t)threadIdx.x;
        if (e < P.n) {
            float4 g, p, m, v = {};
            wt_load<G, OPT>(P, e, g, p, m, v);
            wt_compute_store<OPT>(P, e, g, p, m, v);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) write_record(P);
}

template <typename G>
__global__ void __launch_bounds__(kAdamThreads) adamw_wt_kernel(const AdamParams P) {
    wt_body<G, kOptAdamW>(P);
}

// one tile per iteration, 4 blocks per SM (cm_set_param("adamw_impl", 3))
template <typename G>
__global__ void __launch_bounds__(kAdamThreads, 4) adamw_wt1_kernel(const AdamParams P) {
    wt_body<G, kOptAdamW, false>(P);
}

// SGD-momentum over the same warp tiles: HBM sizeof(G) + 8 read + 8 write B/elem
template <typename G>
__global__ void __launch_bounds__(kAdamThreads) sgd_wt_kernel(const AdamParams P) {
    wt_body<G, kOptSgd>(P);
}

// a bare cross-GPU barrier (cm_barrier): one block meets block 0 of every rank
__global__ void barrier_kernel(const Pads pads, int n, int rank, uint32_t epoch) {
    block_barrier(pads, n, rank, epoch, 0);
}

// the step's scalar record alone (a per-bucket step: the bucket kernels carry no record)
__global__ void record_kernel(const AdamParams P) { write_record(P); }

// ------------------------------------------------------------------ AdamW, TMA-staged
// Same arithmetic as adamw_kernel; data movement by the bulk-copy engine (TMA, 1-D
// cp.async.bulk): one elected thread streams tiles of g, p, m, v into a kTmaStages-deep
// shared-memory ring (mbarrier complete_tx), all threads update p/m/v in shared memory,
// and the same thread bulk-stores the three result tiles.  Few threads, many bytes in
// flight (kTmaStages x tile) per SM, no per-thread address arithmetic on the HBM stream.
constexpr int kTmaThreads = 256;
constexpr int kTmaTile = 4096;          // elements per tile
constexpr int kTmaStages = 3;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(smem_dst)), "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* gmem_dst, const void* smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gmem_dst), "r"(smem_u32(smem_src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <typename G>
struct TmaTile {
    static constexpr int kGBytes = kTmaTile * GT<G>::kBytes;
    static constexpr int kStageBytes = kGBytes + 3 * kTmaTile * 4;
};

template <typename G>
__global__ void __launch_bounds__(kTmaThreads, 1) adamw_tma_kernel(const AdamParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[kTmaStages];
    if (block_nf_blocked(P)) return;
    constexpr int GB = GT<G>::kBytes;
    const int64_t ntiles = (P.n + kTmaTile - 1) / kTmaTile;
    auto stage_ptr = [&](int st) { return smem + (size_t)st * TmaTile<G>::kStageBytes; };
    auto issue = [&](int64_t tile, int st) {
        const int64_t e0 = tile * kTmaTile;
        const int64_t len = (P.n - e0) < kTmaTile ? (P.n - e0) : kTmaTile;
        unsigned char* b = stage_ptr(st);
        const uint32_t gbytes = (uint32_t)(len * GB), fbytes = (uint32_t)(len * 4);
        mbar_expect_tx(&bars[st], gbytes + 3 * fbytes);
        bulk_load(b, (const char*)P.g + e0 * GB, gbytes, &bars[st]);
        bulk_load(b + TmaTile<G>::kGBytes, P.p_in + e0, fbytes, &bars[st]);
        bulk_load(b + TmaTile<G>::kGBytes + kTmaTile * 4, P.m_in + e0, fbytes, &bars[st]);
        bulk_load(b + TmaTile<G>::kGBytes + 2 * kTmaTile * 4, P.v_in + e0, fbytes, &bars[st]);
    };
    const bool leader = threadIdx.x == 0;
    if (leader) {
        for (int st = 0; st < kTmaStages; ++st) mbar_init(&bars[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (leader) {
        for (int st = 0; st < kTmaStages; ++st) {
            const int64_t tile = blockIdx.x + (int64_t)st * gridDim.x;
            if (tile < ntiles) issue(tile, st);
        }
    }
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % kTmaStages;
        const uint32_t phase = (uint32_t)((it / kTmaStages) & 1);
        mbar_wait(&bars[st], phase);
        const int64_t e0 = tile * kTmaTile;
        const int len = (int)((P.n - e0) < kTmaTile ? (P.n - e0) : kTmaTile);
        unsigned char* b = stage_ptr(st);
        float* sp = reinterpret_cast<float*>(b + TmaTile<G>::kGBytes);
        float* sm = sp + kTmaTile;
        float* sv = sm + kTmaTile;
        for (int q = threadIdx.x * 4; q < len; q += kTmaThreads * 4) {
            float4 g;
            if constexpr (std::is_same<G, F32Tag>::value) {
                g = *reinterpret_cast<const float4*>(b + q * 4);
            } else {
                const uint2 w = *reinterpret_cast<const uint2*>(b + q * 2);
                g = make_float4(bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y));
            }
            float4 p = *reinterpret_cast<float4*>(sp + q);
            float4 m = *reinterpret_cast<float4*>(sm + q);
            float4 v = *reinterpret_cast<float4*>(sv + q);
            adamw_elem(g.x, P.s, p.x, m.x, v.x);
            adamw_elem(g.y, P.s, p.y, m.y, v.y);
            adamw_elem(g.z, P.s, p.z, m.z, v.z);
            adamw_elem(g.w, P.s, p.w, m.w, v.w);
            nf_check4(P.nf, P.step, nf_idx(P.nf_base, e0 + q), p, m, v);
            *reinterpret_cast<float4*>(sp + q) = p;
            *reinterpret_cast<float4*>(sm + q) = m;
            *reinterpret_cast<float4*>(sv + q) = v;
        }
        fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the bulk copy
        __syncthreads();
        if (leader) {
            const uint32_t fbytes = (uint32_t)len * 4;
            bulk_store(P.p_out + e0, sp, fbytes);
            bulk_store(P.m_out + e0, sm, fbytes);
            bulk_store(P.v_out + e0, sv, fbytes);
            bulk_commit();
            const int64_t next = tile + (int64_t)kTmaStages * gridDim.x;
            if (next < ntiles) {
                bulk_wait_read0();  // the stores have read this stage; reuse it
                issue(next, st);
            }
        }
    }
    if (leader) bulk_wait0();
    if (blockIdx.x == 0 && threadIdx.x == 0) write_record(P);
}

// ------------------------------------------------------------------ ZeRO-1: AdamW + AG
// SURVEY 8 row f3 (PAPER.md:670-674 discusses sharded optimizers): after the reduce-scatter
// rank r owns the reduced shard r of every bucket (in the tap's HBM staging half).  It
// applies the same AdamW (adamw_elem: identical bits) to its shard only -- m, v are
// shard-local arrays -- and stores each updated parameter once into its own p and once
// into every peer's p over NVLink (the all-gather of the updated parameters, fused into
// the optimizer kernel: no separate collective, no re-read).  Grid-stride over 16-byte
// groups of the shard-local index space; a running bucket index maps j -> flat p index.
struct Zero1Params {
    const void* g;                  // staging half: shard-local reduced gradients
    float* m; float* v;             // shard-local moments
    float* p[kMaxRanks];            // every rank's flat p (index rank = own)
    const BucketDev* buckets;
    int nb, n, rank, barriers;
    int64_t L;                      // shard elements
    AdamScalars s;
    SgdScalars q;
    Pads pads;
    uint32_t epoch;
    volatile float* hp_rec;
    volatile int32_t* hp_kind;
    volatile int64_t* hp_tag;
    float rec[10];
    int32_t rec_kind;
    int64_t step;
    int unroll2;                    // 1: two groups per thread in flight (default), 0: one
    NfRef nf;                       // non-finite report (flat index)
    int64_t j0;                     // first shard-local element (per-bucket step: the bucket's
                                    // shard_off; g then points at shard-local element j0)
};

// shard-local index j -> flat index of rank P.rank's element (b: running bucket index, j
// non-decreasing per thread)
__device__ __forceinline__ int64_t z1_flat(const Zero1Params& P, int64_t j, int& b) {
    while (b + 1 < P.nb && j >= P.buckets[b + 1].shard_off) ++b;
    const BucketDev& B = P.buckets[b];
    return B.off + (int64_t)P.rank * (B.padded / P.n) + (j - B.shard_off);
}
template <typename G, int OPT>
__device__ __forceinline__ void z1_load(const Zero1Params& P, int64_t j, int64_t flat, float4& g, float4& p,
                                        float4& m, float4& v) {
    if constexpr (std::is_same<G, F32Tag>::value) {
        g = __ldcs(reinterpret_cast<const float4*>((const float*)P.g + j));
    } else {
        const uint2 w = __ldcs(reinterpret_cast<const uint2*>((const uint16_t*)P.g + j));
        g = make_float4(bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y));
    }
    p = __ldcs(reinterpret_cast<const float4*>(P.p[P.rank] + flat));
    m = __ldcs(reinterpret_cast<const float4*>(P.m + j));
    if constexpr (OPT == kOptAdamW) v = __ldcs(reinterpret_cast<const float4*>(P.v + j));
}
template <int N, int OPT>
__device__ __forceinline__ void z1_compute_store(const Zero1Params& P, int64_t j, int64_t flat, const float4& g,
                                                 float4 p, float4 m, float4 v) {
    if constexpr (OPT == kOptAdamW) {
        adamw_elem(g.x, P.s, p.x, m.x, v.x);
        adamw_elem(g.y, P.s, p.y, m.y, v.y);
        adamw_elem(g.z, P.s, p.z, m.z, v.z);
        adamw_elem(g.w, P.s, p.w, m.w, v.w);
        __stcs(reinterpret_cast<float4*>(P.v + j), v);
    } else {
        sgd_elem(g.x, P.q, p.x, m.x);
        sgd_elem(g.y, P.q, p.y, m.y);
        sgd_elem(g.z, P.q, p.z, m.z);
        sgd_elem(g.w, P.q, p.w, m.w);
    }
    nf_check4(P.nf, P.step, flat, p, m, v);
    __stcs(reinterpret_cast<float4*>(P.m + j), m);
    const uint4 pw = make_uint4(__float_as_uint(p.x), __float_as_uint(p.y), __float_as_uint(p.z),
                                __float_as_uint(p.w));
#pragma unroll
    for (int k = 0; k < N; ++k) st_v4(P.p[k] + flat, pw);   // own p + all-gather
}

// Grid-stride over 4-element groups of the shard; two groups per thread in flight (their
// loads issued before either is reduced and stored): the kernel's NVLink egress is n-1
// stores per group, and one group of loads per thread left the link under-fed.
template <typename G, int N, int OPT = kOptAdamW>
__global__ void __launch_bounds__(256) adamw_zero1_kernel(Zero1Params P) {
    int b = 0;
    const int64_t groups = P.L / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // shard-local j = P.j0 + 4q; g is indexed relative to j0, m, v, p absolutely
    P.g = (const char*)P.g - P.j0 * GT<G>::kBytes;
    if (P.unroll2) {
        for (; q + stride < groups; q += 2 * stride) {
            const int64_t j0 = P.j0 + q * 4, j1 = P.j0 + (q + stride) * 4;
            const int64_t f0 = z1_flat(P, j0, b), f1 = z1_flat(P, j1, b);
            float4 g0, p0, m0, v0 = {}, g1, p1, m1, v1 = {};
            z1_load<G, OPT>(P, j0, f0, g0, p0, m0, v0);
            z1_load<G, OPT>(P, j1, f1, g1, p1, m1, v1);
            z1_compute_store<N, OPT>(P, j0, f0, g0, p0, m0, v0);
            z1_compute_store<N, OPT>(P, j1, f1, g1, p1, m1, v1);
        }
    }
    for (; q < groups; q += stride) {
        const int64_t j = P.j0 + q * 4;
        const int64_t f = z1_flat(P, j, b);
        float4 g, p, m, v = {};
        z1_load<G, OPT>(P, j, f, g, p, m, v);
        z1_compute_store<N, OPT>(P, j, f, g, p, m, v);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) write_record(P);
    if (P.barriers) block_barrier(P.pads, N, P.rank, P.epoch, 1);   // every shard landed everywhere
}

// ZeRO-1 with the parameter all-gather as bulk copies (cm_set_param("zero1_impl", 2)): the
// updated parameters of a tile go into shared memory, and one elected thread pushes the
// tile to its own p and to every peer's p with n cp.async.bulk stores (the bulk-copy engine
// moves the bytes over NVLink; no per-thread remote stores).  Tiles never straddle a
// bucket, so each tile is one contiguous range of every rank's flat p.  Two tile buffers:
// a buffer is rewritten only after its previous bulk stores have read it.  Same element
// arithmetic (adamw_elem / sgd_elem), same bits.
constexpr int kZ1TmaThreads = 256;
constexpr int kZ1TmaTile = 2048;   // elements: 8 KiB of fp32 parameters

__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

template <typename G, int N, int OPT = kOptAdamW>
__global__ void __launch_bounds__(kZ1TmaThreads) adamw_zero1_tma_kernel(const Zero1Params P) {
    __shared__ __align__(128) float tile[2][kZ1TmaTile];
    const bool leader = threadIdx.x == 0;
    int b = 0;
    int64_t base = 0;   // first tile index of bucket b
    int buf = 0;
    for (int64_t t = blockIdx.x;; t += gridDim.x) {
        int64_t len = 0;
        while (b < P.nb) {
            len = P.buckets[b].padded / P.n;
            const int64_t tb = (len + kZ1TmaTile - 1) / kZ1TmaTile;
            if (t < base + tb) break;
            base += tb;
            ++b;
        }
        if (b >= P.nb) break;
        const BucketDev& B = P.buckets[b];
        const int64_t lo = (t - base) * kZ1TmaTile;
        const int cnt = (int)min((int64_t)kZ1TmaTile, len - lo);          // a multiple of 4
        const int64_t j0 = B.shard_off + lo;                                // shard-local
        const int64_t f0 = B.off + (int64_t)P.rank * len + lo;              // flat
        if (leader) bulk_wait_read1();   // the stores issued from this buffer two tiles ago
        __syncthreads();
        float4 g[2], p[2], m[2], v[2] = {};
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int e = (u * kZ1TmaThreads + threadIdx.x) * 4;
            if (e < cnt) z1_load<G, OPT>(P, j0 + e, f0 + e, g[u], p[u], m[u], v[u]);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int e = (u * kZ1TmaThreads + threadIdx.x) * 4;
            if (e >= cnt) continue;
            if constexpr (OPT == kOptAdamW) {
                adamw_elem(g[u].x, P.s, p[u].x, m[u].x, v[u].x);
                adamw_elem(g[u].y, P.s, p[u].y, m[u].y, v[u].y);
                adamw_elem(g[u].z, P.s, p[u].z, m[u].z, v[u].z);
                adamw_elem(g[u].w, P.s, p[u].w, m[u].w, v[u].w);
                __stcs(reinterpret_cast<float4*>(P.v + j0 + e), v[u]);
            } else {
                sgd_elem(g[u].x, P.q, p[u].x, m[u].x);
                sgd_elem(g[u].y, P.q, p[u].y, m[u].y);
                sgd_elem(g[u].z, P.q, p[u].z, m[u].z);
                sgd_elem(g[u].w, P.q, p[u].w, m[u].w);
            }
            nf_check4(P.nf, P.step, f0 + e, p[u], m[u], v[u]);
            __stcs(reinterpret_cast<float4*>(P.m + j0 + e), m[u]);
            *reinterpret_cast<float4*>(&tile[buf][e]) = p[u];
        }
        fence_proxy_async_smem();        // this thread's smem writes -> visible to the bulk copies
        __syncthreads();
        if (leader) {
#pragma unroll
            for (int k = 0; k < N; ++k) bulk_store(P.p[k] + f0, &tile[buf][0], (uint32_t)cnt * 4u);
            bulk_commit();
        }
        buf ^= 1;
    }
    if (leader) {
        bulk_wait0();                    // every bulk store of this block has completed
        fence_proxy_async_global();      // ... and is ordered before the generic release below
        __threadfence_system();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) write_record(P);
    if (P.barriers) block_barrier(P.pads, N, P.rank, P.epoch, 1);   // every shard landed everywhere
    else __syncthreads();
}

// ------------------------------------------------------------------ shard gather/scatter
// Shard-local index j of rank r <-> flat index off_b + r*E_b/n + (j - shard_off_b).
// dir 0 (snapshot): flat device p/m/v of this rank -> shard-local dst arrays.
// dir 1 (restore):  shard-local src arrays -> flat p/m/v of all ranks (all-gather).
struct ShardCopyParams {
    const float* src[3];
    float* dst[3][kMaxRanks];   // dir 1: per-rank flat buffers; dir 0: [k][0] shard-local
    const BucketDev* buckets;
    int nb, n, rank, dir, barriers;
    int mv_local;               // ZeRO-1: m, v are shard-local arrays of this rank only
    int64_t shard_nvec;         // shard-local 16-byte vectors of fp32
    Pads pads;
    uint32_t epoch;
};

__global__ void __launch_bounds__(256) shard_copy_kernel(const ShardCopyParams P) {
    if (P.dir == 1 && P.barriers) block_barrier(P.pads, P.n, P.rank, P.epoch, 0);
    int b = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < P.shard_nvec;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = q * 4;
        while (b + 1 < P.nb && j >= P.buckets[b + 1].shard_off) ++b;
        const BucketDev B = P.buckets[b];
        const int64_t flat = B.off + (int64_t)P.rank * (B.padded / P.n) + (j - B.shard_off);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const bool local = P.mv_local && a > 0;   // shard-local m/v (ZeRO-1)
            if (P.dir == 0) {
                st_v4(P.dst[a][0] + j, ld_v4(P.src[a] + (local ? j : flat)));
            } else if (local) {
                st_v4(P.dst[a][P.rank] + j, ld_v4(P.src[a] + j));
            } else {
                const uint4 x = ld_v4(P.src[a] + j);
                for (int k = 0; k < P.n; ++k) st_v4(P.dst[a][k] + flat, x);
            }
        }
    }
    if (P.dir == 1 && P.barriers) block_barrier(P.pads, P.n, P.rank, P.epoch, 1);
}

// Bitwise compare of shadow-side shard-local arrays (elements [j0, j0 + len) of the shard,
// sp[0] = element j0) with this rank's training p/m/v.  first_bad = min over mismatches of
// flat * 4 + what (what: 0 p, 1 m, 2 v), so the host learns the first flat index and array.
__global__ void __launch_bounds__(256) compare_kernel(const float* __restrict__ sp, const float* __restrict__ sm,
                                                      const float* __restrict__ sv, const float* __restrict__ p,
                                                      const float* __restrict__ m, const float* __restrict__ v,
                                                      const BucketDev* __restrict__ buckets, int nb, int n,
                                                      int rank, int64_t j0, int64_t len,
                                                      unsigned long long* first_bad, int mv_local) {
    int b = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < len;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = j0 + q;
        while (b + 1 < nb && j >= buckets[b + 1].shard_off) ++b;
        const BucketDev B = buckets[b];
        const int64_t flat = B.off + (int64_t)rank * (B.padded / n) + (j - B.shard_off);
        const int64_t mi = mv_local ? j : flat;
        int what = -1;
        if (__float_as_uint(sv[q]) != __float_as_uint(v[mi])) what = 2;
        if (__float_as_uint(sm[q]) != __float_as_uint(m[mi])) what = 1;
        if (__float_as_uint(sp[q]) != __float_as_uint(p[flat])) what = 0;
        if (what >= 0) atomicMin(first_bad, (unsigned long long)flat * 4ull + (unsigned long long)what);
    }
}

// Bitwise compare of a tap ring slot (shard-local, read through its device alias) with the
// reduced gradients the training step used: the flat grad buffer's shard r (ref_flat = 1) or
// the shard-local staging half (ref_flat = 0, ZeRO-1).  16-byte vectors (a shard is a whole
// number of vectors and 16-byte aligned; the ring is read over PCIe, so the width matters).
// Reports flat * 4 + 3 of the first differing element.
__global__ void __launch_bounds__(256) compare_grads_kernel(const void* ring, const void* ref, int ref_flat,
                                                            const BucketDev* __restrict__ buckets, int nb, int n,
                                                            int rank, int64_t shard_n, int es,
                                                            unsigned long long* first_bad) {
    const int per = 16 / es;                       // elements per vector
    int b = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q * per < shard_n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = q * per;
        while (b + 1 < nb && j >= buckets[b + 1].shard_off) ++b;
        const BucketDev B = buckets[b];
        const int64_t flat = B.off + (int64_t)rank * (B.padded / n) + (j - B.shard_off);
        const int64_t ri = ref_flat ? flat : j;
        const uint4 x = ld_cs_v4((const char*)ring + j * es);
        const uint4 y = ld_v4((const char*)ref + ri * es);
        if (x.x == y.x && x.y == y.y && x.z == y.z && x.w == y.w) continue;
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
        int k = 0;
        for (int w = 0; w < 4; ++w) {
            if (xs[w] == ys[w]) continue;
            k = es == 4 ? w : 2 * w + (((xs[w] ^ ys[w]) & 0xFFFFu) ? 0 : 1);
            break;
        }
        atomicMin(first_bad, (unsigned long long)(flat + k) * 4ull + 3ull);
    }
}

// ------------------------------------------------------------------ low-intensity D2H drain
// A copy engine drains at the host link's full rate, and a saturated device->host link
// delays the GPU's own command fetch: measured, a launch-bound kernel stream runs 17%
// slower next to a 32 GB/s copy-engine drain and not measurably slower next to an 11 GB/s
// single-CTA SM drain (profiles/r01c_interference.md).  With compute to hide under, the
// tap drain and the snapshot persist therefore go through this kernel: `gridDim.x` CTAs
// (1 by default) copy 16-byte vectors from HBM into host-mapped memory with streaming
// stores; the link never saturates, and a few SM slots are the only cost.
__global__ void __launch_bounds__(256) drain_kernel(const uint4* __restrict__ src, uint4* dst, int64_t nvec) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nvec; q += (int64_t)gridDim.x * blockDim.x)
        st_cs_v4(dst + q, ld_cs_v4(src + q));
}

// stream-ordered store of one int64 into host-mapped memory (segment header)
__global__ void publish_kernel(volatile int64_t* dst, int64_t value, const volatile int64_t* skip_nf,
                               int64_t step) {
    if (nf_blocked(skip_nf, step)) return;   // a flagged step is never published
    __threadfence_system();
    *dst = value;
    __threadfence_system();
}

// the same for `count` consecutive tap flags (one coalesced drain of several buckets)
__global__ void publish_range_kernel(volatile uint64_t* dst, int count, uint64_t value) {
    __threadfence_system();
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = value;
    __threadfence_system();
}

// ------------------------------------------------------------------ RS + tap + AG, bulk-copy pipeline
// cm_set_param("ar_impl", 2): the same fused all-reduce with the data movement done by the
// bulk-copy engine (TMA, 1-D cp.async.bulk).  One block per SM walks tiles of the shard; for
// each tile one elected thread pulls the tile from all n ranks' buffers (n-1 of them over
// NVLink) into a shared-memory stage (mbarrier complete_tx), all threads reduce the n copies
// in rank order (reduce_vec: identical bits) into rank 0's slot, and the elected thread pushes
// the result to the tap target and to all n ranks' buffers with bulk stores.  Two stages: the
// next tile's pulls are in flight while this one is reduced and pushed.  Few threads, many
// bytes in flight per SM, no per-thread address arithmetic on the NVLink stream.  Staged tap
// or no tap only (a direct tap keeps the per-thread kernel).
constexpr int kArTmaThreads = 256;
constexpr int kArTmaMaxSmem = 200 * 1024;
template <int N> struct ArTma {
    // default bytes per rank per stage: small tiles keep every SM busy on the mid-size buckets
    // of a training step (measured in the step pattern: n=2 16 MiB 27.2 us with 4 KiB tiles vs
    // 29.8 with 16 KiB; n=4 16 MiB 41.6 us with 4 KiB vs 42.8 with 8 KiB and 44.7 with 12 KiB,
    // GPT-2 lockstep chain 67.3 vs 67.9 us; equal from 64 MiB)
    static constexpr int kTile = 4096;
};

template <typename G, int N, int kArTmaStages>
__global__ void __launch_bounds__(kArTmaThreads, 1) rs_tap_ag_tma_kernel(const ArParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[kArTmaStages];
    const int T = P.tma_tile;
    constexpr int V = GT<G>::kPerVec;
    if (P.pdl_wait) pdl_wait_prior();
    if (P.barriers) block_barrier(P.pads, N, P.rank, P.epoch, 0);   // peers' grads are ready
    pdl_launch_next();
    const int64_t bytes = P.nvec * 16;
    const int64_t ntiles = (bytes + T - 1) / T;
    const bool leader = threadIdx.x == 0;
    auto stage = [&](int st, int k) { return smem + ((size_t)st * N + k) * T; };
    auto issue = [&](int64_t tile, int st) {
        const int64_t off = tile * T;
        const uint32_t len = (uint32_t)((bytes - off) < T ? (bytes - off) : T);
        mbar_expect_tx(&bars[st], len * N);
#pragma unroll
        for (int k = 0; k < N; ++k) bulk_load(stage(st, k), P.buf[k] + off, len, &bars[st]);
    };
    if (leader) {
        for (int st = 0; st < kArTmaStages; ++st) mbar_init(&bars[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (leader)
        for (int st = 0; st < kArTmaStages; ++st) {
            const int64_t tile = blockIdx.x + (int64_t)st * gridDim.x;
            if (tile < ntiles) issue(tile, st);
        }
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % kArTmaStages;
        mbar_wait(&bars[st], (uint32_t)((it / kArTmaStages) & 1));
        const int64_t off = tile * T;
        const int len = (int)((bytes - off) < T ? (bytes - off) : T);
        for (int q = threadIdx.x; q < len / 16; q += kArTmaThreads) {
            uint4 x[N];
#pragma unroll
            for (int k = 0; k < N; ++k) x[k] = *reinterpret_cast<const uint4*>(stage(st, k) + q * 16);
            const uint4 r = reduce_vec<G, N>(x);
            nf_check_vec<G>(P.nf, P.nf_step, P.elem0 + (off / 16 + q) * V, r);
            *reinterpret_cast<uint4*>(stage(st, 0) + q * 16) = r;   // the result replaces rank 0's copy
        }
        fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the bulk stores
        __syncthreads();
        if (leader) {
            if (P.tap) bulk_store(P.tap + off, stage(st, 0), (uint32_t)len);
            if (P.ag) {
#pragma unroll
                for (int k = 0; k < N; ++k) bulk_store(P.buf[k] + off, stage(st, 0), (uint32_t)len);
            }
            bulk_commit();
            const int64_t next = tile + (int64_t)kArTmaStages * gridDim.x;
            if (next < ntiles) {
                bulk_wait_read0();   // the stores have read this stage; refill it
                issue(next, st);
            }
        }
    }
    if (leader) {
        bulk_wait0();                // every bulk store of this block has completed
        fence_proxy_async_global();  // ... and is ordered before the generic releases below
        __threadfence_system();
    }
    __syncthreads();
    ar_epilogue<N>(P);
    pdl_wait_prior();
}

}  // namespace cm
