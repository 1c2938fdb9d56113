// cm_persist.cc -- host-only persistence and serving of the shadow segments (SURVEY 8 row
// f4): CheckpointFile save / load, consolidation, CRC-32-checked
// range serving and the per-tensor model file.  No
// CUDA: these calls work on any process of the host, with or without a GPU or a context.
#include "cm.h"
#include "cm_segment.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

extern "C" {

// ---------------------------------------------------------------- CheckpointFile (f4)
// SPEC.md:371-374 (CheckpointFile, CRC-32 checksum): the host shadow of one
// rank -- snapshot halves, the tapped-gradient ring, step records and flags -- persisted
// to a file and recreated from it (restore then works on another host, or after the
// host's shared memory is gone).  CRC-32 = IEEE 802.3 (reflected 0xEDB88320), the zlib
// checksum, computed slice-by-8.
namespace {
struct FileHeader {
    uint64_t magic;        // kFileMagic
    uint32_t version, crc32;
    uint64_t payload_bytes, layout_hash;
    int32_t world_size, rank;
    int64_t shadow_step;
    uint64_t reserved[2];
};
static_assert(sizeof(FileHeader) == 64, "file header");
constexpr uint64_t kFileMagic = 0x454C49465442434Bull;   // bytes "KCBTFILE"

uint32_t crc_tab[8][256];
void crc_init() {   // once per process; serving threads may call it concurrently
    static std::once_flag once;
    std::call_once(once, [] {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            crc_tab[0][i] = c;
        }
        for (uint32_t i = 0; i < 256; ++i)
            for (int t = 1; t < 8; ++t) crc_tab[t][i] = (crc_tab[t - 1][i] >> 8) ^ crc_tab[0][crc_tab[t - 1][i] & 0xFF];
    });
}
uint32_t crc32_update(uint32_t crc, const unsigned char* p, size_t n) {
    crc = ~crc;
    while (n >= 8) {
        uint32_t a, b;
        memcpy(&a, p, 4);
        memcpy(&b, p + 4, 4);
        a ^= crc;
        crc = crc_tab[7][a & 0xFF] ^ crc_tab[6][(a >> 8) & 0xFF] ^ crc_tab[5][(a >> 16) & 0xFF] ^
              crc_tab[4][a >> 24] ^ crc_tab[3][b & 0xFF] ^ crc_tab[2][(b >> 8) & 0xFF] ^
              crc_tab[1][(b >> 16) & 0xFF] ^ crc_tab[0][b >> 24];
        p += 8;
        n -= 8;
    }
    while (n--) crc = crc_tab[0][(crc ^ *p++) & 0xFF] ^ (crc >> 8);
    return ~crc;
}
}  // namespace

uint32_t cm_crc32(const void* data, size_t n) {
    crc_init();
    return crc32_update(0, (const unsigned char*)data, n);
}

cm_status cm_shadow_save(const char* shm_name, int32_t rank, const char* path) {
    if (!shm_name || !path) return CM_ERR_ARG;
    crc_init();
    char name[256];
    snprintf(name, sizeof name, "/%s.r%d", shm_name, rank);
    int fd = shm_open(name, O_RDONLY, 0);
    if (fd < 0) return CM_ERR_ARG;
    struct stat st;
    if (fstat(fd, &st) != 0 || (size_t)st.st_size < sizeof(SegHeader)) { close(fd); return CM_ERR_ARG; }
    const size_t size = (size_t)st.st_size;
    void* mp = mmap(nullptr, size, PROT_READ, MAP_SHARED, fd, 0);
    close(fd);
    if (mp == MAP_FAILED) return CM_ERR_ARG;
    const SegHeader* h = (const SegHeader*)mp;
    cm_status rc = CM_OK;
    FILE* f = nullptr;
    if (h->magic != kMagic || h->total != size) { rc = CM_ERR_ARG; goto done; }
    {
        FileHeader fh{};
        fh.magic = kFileMagic;
        fh.version = 1;
        fh.payload_bytes = size;
        fh.layout_hash = h->layout_hash;
        fh.world_size = h->world_size;
        fh.rank = h->rank;
        fh.shadow_step = h->shadow_step;
        fh.crc32 = crc32_update(0, (const unsigned char*)mp, size);
        std::string tmp = std::string(path) + ".tmp";
        f = fopen(tmp.c_str(), "wb");
        if (!f) { rc = CM_ERR_ARG; goto done; }
        bool ok = fwrite(&fh, sizeof fh, 1, f) == 1 && fwrite(mp, 1, size, f) == size;
        ok = (fflush(f) == 0) && ok && (fsync(fileno(f)) == 0);
        ok = (fclose(f) == 0) && ok;
        f = nullptr;
        if (!ok || rename(tmp.c_str(), path) != 0) { unlink(tmp.c_str()); rc = CM_ERR_ARG; }
    }
done:
    munmap(mp, size);
    return rc;
}

cm_status cm_shadow_load(const char* path, const char* shm_name, int32_t rank) {
    if (!shm_name || !path) return CM_ERR_ARG;
    crc_init();
    FILE* f = fopen(path, "rb");
    if (!f) return CM_ERR_ARG;
    FileHeader fh{};
    if (fread(&fh, sizeof fh, 1, f) != 1 || fh.magic != kFileMagic || fh.version != 1 || fh.rank != rank ||
        fh.payload_bytes < sizeof(SegHeader) || fh.world_size < 1 || fh.world_size > kSegMaxRanks ||
        fh.rank >= fh.world_size) {
        fclose(f);
        return CM_ERR_ARG;
    }
    // the payload size must be the file's (never trust the header to size a segment), and the
    // segment header inside must describe the same segment before anything is created
    {
        struct stat fs;
        if (fstat(fileno(f), &fs) != 0 || (uint64_t)fs.st_size != sizeof(FileHeader) + fh.payload_bytes) {
            fclose(f);
            return CM_ERR_ARG;
        }
        SegHeader sh{};
        if (fread(&sh, sizeof sh, 1, f) != 1 || sh.magic != kMagic || sh.version != kVersion ||
            sh.total != fh.payload_bytes || sh.rank != rank || sh.world_size != fh.world_size ||
            sh.layout_hash != fh.layout_hash) {
            fclose(f);
            return CM_ERR_INVARIANT;
        }
        if (fseek(f, (long)sizeof fh, SEEK_SET) != 0) {
            fclose(f);
            return CM_ERR_ARG;
        }
    }
    char name[256];
    snprintf(name, sizeof name, "/%s.r%d", shm_name, rank);
    shm_unlink(name);
    int fd = shm_open(name, O_RDWR | O_CREAT | O_EXCL, 0600);
    if (fd < 0) { fclose(f); return CM_ERR_ARG; }
    cm_status rc = CM_OK;
    void* mp = MAP_FAILED;
    if (ftruncate(fd, (off_t)fh.payload_bytes) != 0) rc = CM_ERR_ARG;
    if (rc == CM_OK) mp = mmap(nullptr, fh.payload_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (mp == MAP_FAILED) rc = CM_ERR_ARG;
    if (rc == CM_OK && fread(mp, 1, fh.payload_bytes, f) != fh.payload_bytes) rc = CM_ERR_ARG;
    if (rc == CM_OK && crc32_update(0, (const unsigned char*)mp, fh.payload_bytes) != fh.crc32)
        rc = CM_ERR_INVARIANT;   // corrupted checkpoint: refuse it
    if (rc == CM_OK && ((const SegHeader*)mp)->layout_hash != fh.layout_hash) rc = CM_ERR_INVARIANT;
    if (mp != MAP_FAILED) munmap(mp, fh.payload_bytes);
    fclose(f);
    if (rc != CM_OK) shm_unlink(name);
    return rc;
}

// ---------------------------------------------------------------- shadow serving (f4)
// SPEC.md:422-430 serve_checkpoint, SPEC.md:411-421 consolidate.  A
// read-only mapping of a live (or loaded) host segment: any process on the host serves.
namespace {
struct SegView {
    void* mp = MAP_FAILED;
    size_t size = 0;
    const SegHeader* h = nullptr;
    SegView() = default;
    SegView(const SegView&) = delete;
    SegView& operator=(const SegView&) = delete;
    ~SegView() { if (mp != MAP_FAILED) munmap(mp, size); }
    // open rank `rank`'s segment read-only and check that it is one of ours with host halves
    cm_status open(const char* shm_name, int32_t rank) {
        if (!shm_name || rank < 0) return CM_ERR_ARG;
        char name[256];
        snprintf(name, sizeof name, "/%s.r%d", shm_name, rank);
        int fd = shm_open(name, O_RDONLY, 0);
        if (fd < 0) return CM_ERR_ARG;
        struct stat st;
        if (fstat(fd, &st) != 0 || (size_t)st.st_size < sizeof(SegHeader)) { close(fd); return CM_ERR_ARG; }
        size = (size_t)st.st_size;
        mp = mmap(nullptr, size, PROT_READ, MAP_SHARED, fd, 0);
        close(fd);
        if (mp == MAP_FAILED) return CM_ERR_ARG;
        h = (const SegHeader*)mp;
        if (h->magic != kMagic || h->version != kVersion || h->total != size || h->rank != rank ||
            h->shadow_place != CM_SHADOW_HOST || h->shard_numel < 0 ||
            h->state_off + 6 * (uint64_t)h->shard_numel * 4 > size)
            return CM_ERR_ARG;
        return CM_OK;
    }
    int64_t half(int i) const {
        return __atomic_load_n((const int64_t*)&h->half_step[i], __ATOMIC_ACQUIRE);
    }
    int64_t newest() const { return std::max(half(0), half(1)); }
    const float* array(int hf, int what) const {
        return (const float*)((const char*)mp + h->state_off) + ((size_t)hf * 3 + what) * h->shard_numel;
    }
};
}  // namespace

cm_status cm_shadow_query(const char* shm_name, int32_t rank, cm_shadow_desc* out) {
    if (!out) return CM_ERR_ARG;
    SegView s;
    cm_status st = s.open(shm_name, rank);
    if (st != CM_OK) return st;
    memset(out, 0, sizeof *out);
    out->world_size = s.h->world_size;
    out->rank = s.h->rank;
    out->dtype = s.h->dtype;
    out->ring_depth = s.h->ring_depth;
    out->n_buckets = s.h->n_buckets;
    out->shard_numel = s.h->shard_numel;
    out->layout_hash = s.h->layout_hash;
    out->shadow_step = s.h->shadow_step;
    out->half_step[0] = s.half(0);
    out->half_step[1] = s.half(1);
    out->nf_step = s.h->nf_step;
    return CM_OK;
}

cm_status cm_shadow_consolidate(const char* shm_name, int32_t world_size, int64_t* step_out) {
    if (!shm_name || !step_out || world_size < 1 || world_size > kSegMaxRanks) return CM_ERR_ARG;
    std::vector<SegView> v(world_size);
    int64_t I = INT64_MAX;
    for (int r = 0; r < world_size; ++r) {
        cm_status st = v[r].open(shm_name, r);
        if (st != CM_OK) return st;
        if (v[r].h->world_size != world_size || v[r].h->layout_hash != v[0].h->layout_hash) return CM_ERR_CONFIG;
        I = std::min(I, v[r].newest());
    }
    if (I < 0) return CM_ERR_STATE;                   // some shard holds no snapshot at all
    for (int r = 0; r < world_size; ++r)
        if (v[r].half(0) != I && v[r].half(1) != I) return CM_ERR_STATE;   // advanced past I twice
    *step_out = I;
    return CM_OK;
}

cm_status cm_shadow_serve(const char* shm_name, int32_t rank, int64_t step, int32_t what, int64_t off,
                          int64_t count, void* dst, uint32_t* crc_out) {
    if (what < 0 || what > 2 || off < 0 || count < 0 || (count > 0 && !dst)) return CM_ERR_ARG;
    SegView s;
    cm_status st = s.open(shm_name, rank);
    if (st != CM_OK) return st;
    if (off > s.h->shard_numel || count > s.h->shard_numel - off) return CM_ERR_ARG;   // outside the shard
    if (step < 0) return CM_ERR_STATE;
    const int hf = s.half(0) == step ? 0 : s.half(1) == step ? 1 : -1;
    if (hf < 0) return CM_ERR_STATE;
    memcpy(dst, s.array(hf, what) + off, (size_t)count * 4);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    if (s.half(hf) != step) return CM_ERR_STATE;    // rewritten while we copied: torn
    if (crc_out) {
        crc_init();
        *crc_out = crc32_update(0, (const unsigned char*)dst, (size_t)count * 4);
    }
    return CM_OK;
}

// Model checkpoint file (SPEC.md:371-374 CheckpointFile: per-layer records + checksum;
// SPEC.md:430 "reassembled model equals consolidated checkpoint"): the consolidated step
// gathered from the n shards into per-tensor records in the caller's tensor order.
namespace {
struct ModelFileHeader {
    uint64_t magic;          // kModelMagic
    uint32_t version;        // 1
    int32_t n_tensors, world_size, dtype;
    int64_t step;
    uint64_t layout_hash;
    int64_t cap_bytes;
    uint32_t crc32;          // of every byte after this header
    uint32_t pad[3];
};
static_assert(sizeof(ModelFileHeader) == 64, "model file header");
struct TensorRecord {        // followed by p, m, v: numel fp32 each
    int64_t index, numel;
    uint32_t crc32[3];       // of p, m, v
    uint32_t pad;
};
static_assert(sizeof(TensorRecord) == 32, "tensor record");
constexpr uint64_t kModelMagic = 0x4C444F4D5442434Bull;   // bytes "KCBTMODL"
}  // namespace

cm_status cm_shadow_export(const char* shm_name, const cm_layer_table* t, int32_t world_size, int64_t step,
                           const char* path, int64_t* step_out) {
    if (!shm_name || !t || !t->numel || !path || world_size < 1 || world_size > kSegMaxRanks) return CM_ERR_ARG;
    if (t->grad_dtype != CM_F32 && t->grad_dtype != CM_BF16) return CM_ERR_CONFIG;
    // the run's plan, through the public planner (cm_plan_buckets / cm_plan_bucket_table)
    std::vector<int64_t> tensor_off(t->n_tensors > 0 ? t->n_tensors : 1);
    int64_t padded = 0;
    int32_t nb = 0;
    if (cm_plan_buckets(t, world_size, &padded, &nb, tensor_off.data()) != CM_OK) return CM_ERR_CONFIG;
    std::vector<int64_t> b_off(nb), b_pad(nb);
    if (cm_plan_bucket_table(t, world_size, nb, b_off.data(), b_pad.data(), nullptr, &nb) != CM_OK)
        return CM_ERR_CONFIG;
    const std::vector<int64_t> numel(t->numel, t->numel + t->n_tensors);
    const uint64_t lh = layout_hash_of(numel, t->cap_bytes, t->grad_dtype, world_size);
    if (step < 0) {
        cm_status st = cm_shadow_consolidate(shm_name, world_size, &step);
        if (st != CM_OK) return st;
    }
    std::vector<SegView> seg(world_size);
    std::vector<int> hf(world_size);
    for (int r = 0; r < world_size; ++r) {
        cm_status st = seg[r].open(shm_name, r);
        if (st != CM_OK) return st;
        if (seg[r].h->world_size != world_size || seg[r].h->layout_hash != lh ||
            seg[r].h->shard_numel != padded / world_size)
            return CM_ERR_CONFIG;
        hf[r] = seg[r].half(0) == step ? 0 : seg[r].half(1) == step ? 1 : -1;
        if (hf[r] < 0) return CM_ERR_STATE;
    }
    crc_init();
    const std::string tmp = std::string(path) + ".tmp";
    FILE* f = fopen(tmp.c_str(), "wb");
    if (!f) return CM_ERR_ARG;
    ModelFileHeader fh{};
    fh.magic = kModelMagic;
    fh.version = 1;
    fh.n_tensors = t->n_tensors;
    fh.world_size = world_size;
    fh.dtype = t->grad_dtype;
    fh.step = step;
    fh.layout_hash = lh;
    fh.cap_bytes = t->cap_bytes;
    bool ok = fwrite(&fh, sizeof fh, 1, f) == 1;
    uint32_t crc = 0;
    std::vector<float> buf;
    // bucket of each tensor (the planner's tensors of one bucket are contiguous in it)
    std::vector<int> bucket_of(t->n_tensors, 0);
    for (int b = 0; b < nb; ++b)
        for (int i = 0; i < t->n_tensors; ++i)
            if (tensor_off[i] >= b_off[b] && tensor_off[i] < b_off[b] + b_pad[b]) bucket_of[i] = b;
    for (int i = 0; ok && i < t->n_tensors; ++i) {
        const int64_t B_off = b_off[bucket_of[i]], B_pad = b_pad[bucket_of[i]];
        const int64_t s = B_pad / world_size, lo = tensor_off[i], hi = lo + numel[i];
        TensorRecord rec{};
        rec.index = i;
        rec.numel = numel[i];
        buf.resize((size_t)numel[i] * 3);
        for (int w = 0; w < 3; ++w) {
            float* dst = buf.data() + (size_t)w * numel[i];
            for (int r = 0; r < world_size; ++r) {   // the pieces of [lo, hi) rank r owns
                const int64_t a = std::max(lo, B_off + r * s), e = std::min(hi, B_off + (r + 1) * s);
                if (a < e)   // shard r of the bucket sits at B_off / n in rank r's shard-local arrays
                    memcpy(dst + (a - lo), seg[r].array(hf[r], w) + B_off / world_size + (a - B_off - r * s),
                           (size_t)(e - a) * 4);
            }
            rec.crc32[w] = crc32_update(0, (const unsigned char*)dst, (size_t)numel[i] * 4);
        }
        crc = crc32_update(crc, (const unsigned char*)&rec, sizeof rec);
        crc = crc32_update(crc, (const unsigned char*)buf.data(), buf.size() * 4);
        ok = fwrite(&rec, sizeof rec, 1, f) == 1 && fwrite(buf.data(), 4, buf.size(), f) == buf.size();
    }
    // every half still holds `step`: nothing was rewritten under the copies (seqlock)
    std::atomic_thread_fence(std::memory_order_seq_cst);
    bool torn = false;
    for (int r = 0; r < world_size; ++r) torn = torn || seg[r].half(hf[r]) != step;
    fh.crc32 = crc;
    ok = ok && fseek(f, 0, SEEK_SET) == 0 && fwrite(&fh, sizeof fh, 1, f) == 1;
    ok = (fflush(f) == 0) && ok && (fsync(fileno(f)) == 0);
    ok = (fclose(f) == 0) && ok;
    if (!ok || torn || rename(tmp.c_str(), path) != 0) {
        unlink(tmp.c_str());
        return torn ? CM_ERR_STATE : CM_ERR_ARG;
    }
    if (step_out) *step_out = step;
    return CM_OK;
}

cm_status cm_unlink_shadow(const char* name, int32_t rank) {
    if (!name) return CM_ERR_ARG;
    char buf[256];
    snprintf(buf, sizeof buf, "/%s.r%d", name, rank);
    return shm_unlink(buf) == 0 ? CM_OK : CM_ERR_ARG;
}

}  // extern "C"
