// cm_segment.h -- the host shadow segment's layout, shared by the device runtime
// (cm_runtime.cu) and the host-only persistence / serving code (cm_persist.cc).  Internal:
// not part of the C ABI (include/cm.h).
//
// One POSIX shm segment per rank: "/<name>.r<rank>".
//   [0, 4096)          SegHeader
//   slot meta          D x SlotMeta (the step scalars recorded for the shadow / roll-forward)
//   flags              D x n_buckets x uint64 (tap flag: iteration+1 once the shard is in)
//   ring               D x shard_numel x sizeof(G)    (the tap ring, shard-local layout)
//   state (HOST)       2 halves x {p, m, v} x shard_numel fp32 (ping-pong shadow state)
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace {

constexpr int kSegMaxRanks = 8;                  // = cm::kMaxRanks
constexpr uint64_t kMagic = 0x434B4D5442323030ull;  // "CKMTB200"
constexpr uint32_t kVersion = 2;   // 2: non-finite report in the header
constexpr size_t kAlign = 4096;

struct SegHeader {
    uint64_t magic;
    uint32_t version;
    int32_t world_size, rank, dtype, ring_depth, n_buckets, shadow_place, pad0;
    int64_t shard_numel;
    uint64_t layout_hash;
    volatile int64_t shadow_step;   // last step published by the shadow
    volatile int64_t half_step[2];  // step held by each ping-pong half, -1 = invalid
    uint64_t meta_off, flags_off, ring_off, state_off, total;
    // non-finite report (written by the kernels through the device alias): the first step
    // whose reduced gradients or updated state held an inf/NaN, and a flat element index
    // (-1: unknown).  -1 = none.  Restore never rolls forward to or past nf_step.
    volatile int64_t nf_step, nf_index;
};
static_assert(sizeof(SegHeader) <= kAlign, "header");

struct SlotMeta {
    volatile int64_t step_tag;  // step whose scalars follow (written after them)
    volatile float sc[10];      // AdamScalars (kind 0) or SgdScalars (kind 1)
    volatile int32_t kind;      // OptKind of the step
    int32_t pad[3];
};
static_assert(sizeof(SlotMeta) == 64, "meta");

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < n; ++i) { h ^= p[i]; h *= 0x100000001B3ull; }
    return h;
}

// The layout a segment was built for: tensor sizes, bucket cap, gradient dtype, n.
inline uint64_t layout_hash_of(const std::vector<int64_t>& numel, int64_t cap_bytes, int32_t dtype, int32_t n) {
    uint64_t h = 0xCBF29CE484222325ull;
    h = fnv1a(h, numel.data(), numel.size() * sizeof(int64_t));
    h = fnv1a(h, &cap_bytes, sizeof cap_bytes);
    h = fnv1a(h, &dtype, sizeof dtype);
    h = fnv1a(h, &n, sizeof n);
    return h;
}

}  // namespace
