/*
 * cm.h -- C ABI of libcm.so: the B200-native hot path of Checkmate (arXiv 2507.13522).
 *
 * The path: a per-iteration bucketed gradient all-reduce across the GPUs
 * of one NVSwitch box whose reduced result is also "multicast" -- tapped exactly once
 * into a pinned, host-mapped shadow ring -- plus the deterministic AdamW step that the
 * training replica applies and that a shadow replica re-applies off the critical path,
 * plus a restore path that rebuilds training state from the shadow.
 *
 *   PAPER.md:32 (sec 1)  "model updates are deterministic: given a model state at time t
 *                         and its corresponding gradients, applying the optimizer step
 *                         produces the state at time t+1"
 *   PAPER.md:35          "replicates reduced gradients ... multicasts them to shadow nodes,
 *                         which apply these updates to independently maintained replicas"
 *
 * Conventions for every call:
 *   - Plain C types only.  `stream` arguments are cudaStream_t handles passed as void*
 *     (NULL = the legacy default stream).  Device pointers are CUDA device addresses on
 *     the context's device; host pointers are ordinary process addresses.
 *   - No exception crosses the ABI.  Every call returns a cm_status; on failure a
 *     message is available from cm_last_error(ctx).  CM_ERR_CUDA is sticky: once a CUDA
 *     call failed the context refuses further work.
 *   - Enqueueing calls (allreduce, apply, shadow apply, gen, restore) are asynchronous
 *     with respect to the host: they enqueue kernels on `stream` and return.  Device-side
 *     faults surface at the next call that synchronises.
 *   - Thread safety: one context is driven by one host thread at a time.
 *   - The library never falls back to a CPU implementation: without a usable CUDA
 *     device cm_init fails with CM_ERR_CUDA.
 *   - Non-finite values ("non-finite input -> numeric error"; reading R16):
 *     the all-reduce kernels check every reduced value and the optimizer kernels every
 *     updated p/m/v.  An inf/NaN is reported into the segment header (step, flat index): the
 *     shadow never applies or publishes that step and restore never rolls forward to it.
 *     The error is CM_ERR_INVARIANT from cm_check (no synchronisation) and cm_verify_ex
 *     (synchronising) until cm_restore rolls back to the last finite step.  Collective calls
 *     do not refuse on it: ranks see the report at different times, and one rank refusing a
 *     collective its peers issued would leave their kernels at a barrier.  Poll cm_check and
 *     agree across ranks (like a loss scaler's found-inf) before calling cm_restore.
 */
#ifndef CM_H_
#define CM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cm_ctx cm_ctx; /* opaque; one per GPU rank (or per virtual rank) */

/* Status codes.  0/2/3/4 follow SPEC.md:616 (ok / config / invariant / unrecoverable). */
typedef enum {
    CM_OK = 0,
    CM_ERR_ARG = 1,           /* null / misaligned pointer, index out of range             */
    CM_ERR_CONFIG = 2,        /* bad world size, ring depth, layer table, no peer access   */
    CM_ERR_INVARIANT = 3,     /* verification mismatch (shadow != train), non-finite state */
    CM_ERR_UNRECOVERABLE = 4, /* no consistent shadow step to restore from                 */
    CM_ERR_CUDA = 5,          /* a CUDA call failed (sticky)                               */
    CM_ERR_STATE = 6          /* call out of order: iteration gap, partial iteration,
                                 layout mismatch, ring slot not released                   */
} cm_status;

typedef enum { CM_F32 = 0, CM_BF16 = 1 } cm_dtype; /* gradient dtype; state is always fp32 */

/* Where the shadow replica's (p, m, v) lives.  The tap ring is host memory in both cases
 * (north_star: "streams each reduced shard once into a pinned, host-mapped shadow ring").
 *   HOST:   POSIX shared memory, survives the training process and the GPU (the analog of
 *           the paper's separate CPU shadow cluster).
 *   DEVICE: a library-owned HBM allocation outside the training buffers; survives only an
 *           in-process ("soft") failure.  Arithmetic is identical in both placements.   */
typedef enum { CM_SHADOW_HOST = 0, CM_SHADOW_DEVICE = 1 } cm_shadow_place;

/* cm_config.flags */
#define CM_FLAG_NO_TAP (1ull << 0)    /* all-reduce + AdamW only: no tap, no shadow (the
                                         "no checkpoint" arm run on our own kernels)       */
#define CM_FLAG_ATTACH (1ull << 1)    /* attach to an existing shadow segment (restart
                                         after a failure) instead of creating a fresh one  */
/* The tap (how each reduced shard reaches the host ring exactly once).  Default, "staged":
 * the fused RS+AG kernel also stores the reduced registers into an HBM staging half (no
 * re-read of the grad buffer), and a copy engine drains the staging half to the pinned
 * host ring off the training stream, so no SM ever waits on PCIe and the grad buffer is
 * free when the kernel ends.  Measured best: GPT-2 model mode at n=1
 * +1.2% iteration time for the tap vs +8.3% direct, +3.1% copy-engine.                  */
#define CM_FLAG_TAP_COPYENGINE (1ull << 2) /* ablation: the copy engine reads the reduced
                                         shard back from the grad buffer after the kernel;
                                         cm_apply_step then waits for those copies       */
#define CM_FLAG_TAP_DIRECT (1ull << 4) /* the kernel stores the reduced registers straight into
                                         the pinned host ring (zero extra HBM traffic; the
                                         kernel then runs at host-link speed)               */
#define CM_FLAG_ZERO1 (1ull << 5)      /* sharded optimizer state (ZeRO-1, SURVEY 8 row f3,
                                         PAPER.md:670-674): the kernel reduce-scatters (no
                                         gradient all-gather); cm_apply_step runs AdamW on
                                         this rank's shard only and all-gathers the updated
                                         parameters over NVLink in the same kernel.  m and v
                                         passed to cm_register_buckets are then shard-local
                                         arrays of P_pad/n elements.  Bit-identical to the
                                         unsharded path (same element arithmetic).         */
#define CM_FLAG_NVLS (1ull << 6)       /* small buckets (the one-shot push kernel, SURVEY 8 row
                                         f2, "PRE" multicast analog): each
                                         rank pushes its bucket ONCE with multimem.st into an
                                         NVLink-SHARP multicast inbox and the NVSwitch
                                         replicates it to all n ranks (egress S_b instead of
                                         (n-1) S_b).  cm_connect creates the multicast object
                                         (rank 0) and hands it to the peers over a local Unix
                                         socket; CM_ERR_CONFIG if the box has no multicast
                                         support.  Multi-process ranks only.  Same bits.    */
#define CM_FLAG_OVERWRITE (1ull << 7) /* create the shadow segment even if one of that name exists
                                         (it is deleted first).  Without it, cm_connect refuses
                                         (CM_ERR_STATE) to replace a surviving segment: after a
                                         hard kill it is the only restore source (attach it with
                                         CM_FLAG_ATTACH instead)                            */
#define CM_FLAG_NO_SHADOW (1ull << 3) /* benchmark mode (bucket sweep): tap into the ring but
                                         keep no shadow replica and no flow control; the ring
                                         is overwritten freely; shadow/verify/restore refuse */

typedef struct {
    int32_t world_size;   /* n, 1..8: data-parallel ranks on this box                      */
    int32_t rank;         /* r, 0..n-1                                                      */
    int32_t device;       /* CUDA device ordinal this rank uses                             */
    int32_t ring_depth;   /* D >= 2: iterations the tap ring holds (flow-control window)    */
    int32_t shadow_place; /* cm_shadow_place                                                */
    int32_t persist_every;/* K (HOST placement): persist a host snapshot of the shadow state
                             every K steps (0/1 = every step).  Every step stays recoverable
                             from host memory alone: restore rolls forward over the tapped
                             gradients since the snapshot, so the host link carries 12/K
                             instead of 12 B/element of state per step.  1 <= K <= D.
                             Ranks in separate processes: K >= 2 (0/1 become 2) and
                             D >= K + 1, else cm_connect fails with CM_ERR_CONFIG -- a hard
                             kill can leave a peer's durable log up to two steps behind, and
                             every shard must still reach that step.         */
    const char *shm_name; /* base name of the shadow segment; rank r uses "/<name>.r<r>".
                             Required unless CM_FLAG_NO_TAP.  Copied by cm_init.            */
    uint64_t flags;       /* CM_FLAG_*                                                      */
} cm_config;

/* The model's parameter tensors in model order ("bin-packing them, starting
 * from the last model layer and working backwards").  numel[i] > 0.       */
typedef struct {
    const int64_t *numel;
    int32_t n_tensors;
    int32_t grad_dtype; /* cm_dtype */
    int64_t cap_bytes;  /* bucket cap in bytes of the gradient dtype; 25 MiB in DDP     */
} cm_layer_table;

/* AdamW hyper-parameters for one step (defaults).  The
 * caller's learning-rate schedule passes lr for the step (PAPER.md:496 uses cosine
 * annealing); the library records it so the shadow applies identical bits (reading R8). */
typedef struct {
    double lr, beta1, beta2, eps, weight_decay;
} cm_adamw;

/* SGD-with-momentum hyper-parameters for one step (SPEC.md:310-316
 * [OP] sgd_step; PAPER.md:307 names SGD among the functional optimizers).  weight_decay
 * != 0 adds the coupled L2 term to the gradient (reading R27); 0 gives the SPEC form. */
typedef struct {
    double lr, momentum, weight_decay;
} cm_sgd;

/* ------------------------------------------------------------------ planning (pure)
 * cm_plan_buckets -- the bucket plan, PAPER.md:258-264 (sec 4.2.2), reading R10-R13:
 * walk tensors from the last to the first; add a tensor to the open bucket while the
 * bucket's bytes stay <= cap_bytes; a tensor larger than cap gets a dedicated bucket
 * (closing the open one).  Each bucket is zero-padded to a multiple of n*V elements,
 * V = 16 B / sizeof(grad), so it splits into n equal 16-byte-aligned shards.
 * The flat layout is bucket 0 first; inside a bucket the tensors in the order added.
 *   out_padded_numel   total flat elements P_pad (size every flat buffer to this)
 *   out_n_buckets      number of buckets
 *   tensor_elem_offset optional [n_tensors]: flat element offset of each tensor
 * Host-only, no device needed.  CM_ERR_CONFIG on an empty/invalid table.            */
cm_status cm_plan_buckets(const cm_layer_table *table, int32_t world_size,
                          int64_t *out_padded_numel, int32_t *out_n_buckets,
                          int64_t *tensor_elem_offset);

/* cm_plan_bucket_table -- the same plan as a table: for bucket b its flat element offset
 * off[b], padded length E_b = padded[b] and real elements used[b] (arrays of `capacity`
 * entries, any may be NULL).  Rank r owns shard [off + r E_b/n, off + (r+1) E_b/n) of every
 * bucket.  *out_n_buckets is always set; CM_ERR_ARG if capacity is too small.
 * Host-only.                                                                            */
cm_status cm_plan_bucket_table(const cm_layer_table *table, int32_t world_size, int32_t capacity, int64_t *off,
                               int64_t *padded, int64_t *used, int32_t *out_n_buckets);

/* ------------------------------------------------------------------ lifecycle
 * cm_init -- create a context for one rank: select the device, allocate the signal pad
 * used by the cross-GPU barriers.  CM_ERR_CONFIG for n outside 1..8, rank outside
 * [0,n), D < 2; CM_ERR_CUDA if the device cannot be used.                             */
cm_status cm_init(const cm_config *cfg, cm_ctx **out);

/* cm_register_buckets -- plan the buckets and register the caller's flat buffers.
 *   grad   device, P_pad elements of grad_dtype: this rank's gradients in the flat
 *          layout; after cm_allreduce_multicast of bucket b it holds the reduced SUM.
 *   p,m,v  device, P_pad fp32 each: master weights and AdamW moments (flat layout).
 *          With CM_FLAG_ZERO1, m and v hold P_pad/n elements: this rank's shard, in the
 *          shard-local order (shard r of bucket b at offset off_b/n).
 * All four must be 16-byte aligned, must outlive the context, and are owned by the
 * caller.  Writes an opaque exchange blob (this rank's IPC handles) into blob_out; on
 * entry *blob_len is its capacity (cm_blob_size() bytes suffice), on exit its length.
 * CM_ERR_ARG for null/misaligned pointers; CM_ERR_CONFIG for a bad table.             */
cm_status cm_register_buckets(cm_ctx *ctx, const cm_layer_table *table, void *grad,
                              float *p, float *m, float *v, void *blob_out, size_t *blob_len);
size_t cm_blob_size(void);

/* cm_connect -- collective over the n ranks (each calls it with everyone's blobs, in
 * rank order, concatenated: n * blob_len bytes, e.g. from torch all_gather_object).
 * Maps the peers' buffers and signal pads (CUDA IPC over NVLink; in-process peers --
 * "virtual ranks" on one GPU -- are used directly and need no barriers), creates (or
 * with CM_FLAG_ATTACH attaches) the shadow segment, and -- when creating -- copies the
 * step-0 state shard r into the shadow (reading R19, "a prior checkpoint
 * replica").  Blocks until that copy is done.  CM_ERR_CONFIG if the blobs disagree on
 * n / layout or a peer is not reachable; CM_ERR_STATE if an attached segment's layout
 * differs.                                                              */
cm_status cm_connect(cm_ctx *ctx, const void *peer_blobs, size_t blob_len);

/* cm_finalize -- synchronise, unmap peers and the segment, free library memory.  The
 * shadow segment is NOT unlinked (it is the restore source); see cm_unlink_shadow.     */
cm_status cm_finalize(cm_ctx *ctx);
cm_status cm_unlink_shadow(const char *shm_name, int32_t rank);

/* Shadow persistence (SPEC.md:371-374 CheckpointFile, SPEC.md:446
 * CRC-32).  Host-only, no device or context needed.
 * cm_shadow_save -- write rank `rank`'s shadow segment (snapshot halves, tapped-gradient
 *   ring, step records, tap flags: everything restore needs) to `path` as a
 *   CheckpointFile: a 64-byte header (magic, version, CRC-32 of the payload, payload
 *   bytes, layout hash, world size, rank, shadow step) + the segment bytes.  Written to
 *   `path`.tmp, fsync'd, renamed.  Call it while the segment is quiescent (after cm_join
 *   and a stream sync, or after the trainer died).  CM_ERR_ARG if the segment is missing.
 * cm_shadow_load -- verify a CheckpointFile (magic, rank, size, CRC-32, layout hash) and
 *   recreate the shm segment from it; a context created with CM_FLAG_ATTACH then restores
 *   from it (e.g. on a new host).  CM_ERR_INVARIANT if the CRC or layout does not match
 *   (the segment is not created), CM_ERR_ARG for an unreadable / malformed file.
 * cm_crc32 -- the checksum used (IEEE 802.3 / zlib CRC-32), exposed for tests.          */
cm_status cm_shadow_save(const char *shm_name, int32_t rank, const char *path);
cm_status cm_shadow_load(const char *path, const char *shm_name, int32_t rank);
uint32_t cm_crc32(const void *data, size_t n);

/* Shadow serving (SPEC.md:422-430 serve_checkpoint, SPEC.md:411-421
 * consolidate; sec 4.2.4 "each shadow node serves as a checkpoint to
 * the training nodes simultaneously").  Host-only, no device or context: any process on
 * the host may serve a live segment while training runs.  Only HOST-placed shadows hold
 * host snapshot halves; a segment without them is CM_ERR_ARG.
 * cm_shadow_query -- describe rank `rank`'s segment: layout, and the step held by each
 *   snapshot half (-1 = invalid or being rewritten).  CM_ERR_ARG if the segment is missing
 *   or malformed.
 * cm_shadow_consolidate -- I = min over ranks 0..world_size-1 of the newest snapshot step
 *   each shard holds (SPEC.md:413-416 min rule); every shard must still hold I in one of
 *   its two halves (the retained previous half), else CM_ERR_STATE
 *   ("consolidation failure").  All segments must agree on world size and layout hash
 *   (CM_ERR_CONFIG).  *step_out = I.
 * cm_shadow_serve -- copy elements [off, off+count) of the shard-local fp32 array `what`
 *   (0 p, 1 m, 2 v; shard-local order: shard r of bucket b at element off_b/n, see
 *   cm_plan_bucket_table) at step `step` from the snapshot half that holds it into the
 *   caller's host buffer dst (count*4 bytes, any alignment), and return the IEEE CRC-32 of
 *   the bytes served in *crc_out (may be NULL).  The half's step word is read before and
 *   after the copy (the shadow sets it to -1 before rewriting a half): if it changed, the
 *   bytes may be torn and the call returns CM_ERR_STATE (retry at a newer consolidated
 *   step).  CM_ERR_ARG for a range outside the owned shard (off < 0, count < 0,
 *   off+count > shard_numel), a bad `what`, or a missing segment; CM_ERR_STATE if no half
 *   holds `step`.  count = 0 serves nothing (CRC of no bytes = 0).                     */
typedef struct {
    int32_t world_size, rank, dtype, ring_depth, n_buckets, pad0;
    int64_t shard_numel;      /* elements of this rank's shard (sum of E_b / n)           */
    uint64_t layout_hash;
    int64_t shadow_step;      /* last step the shadow published                          */
    int64_t half_step[2];     /* step held by each host snapshot half, -1 = invalid      */
    int64_t nf_step;          /* first non-finite step reported, -1 = none               */
} cm_shadow_desc;
cm_status cm_shadow_query(const char *shm_name, int32_t rank, cm_shadow_desc *out);
cm_status cm_shadow_consolidate(const char *shm_name, int32_t world_size, int64_t *step_out);
cm_status cm_shadow_serve(const char *shm_name, int32_t rank, int64_t step, int32_t what, int64_t off,
                          int64_t count, void *dst, uint32_t *crc_out);

/* cm_shadow_export -- write the checkpoint at `step` (step < 0: the consolidated step) of
 * the n = world_size shards to `path` as a model file with per-tensor records (SPEC.md:
 * 371-374 CheckpointFile: per-layer + optimizer records, checksum; SPEC.md:430 the
 * reassembled model equals the consolidated checkpoint), in the tensor order of `table`
 * (the table the run registered; its plan must match the segments' layout hash).
 * Little-endian, no padding:
 *   header (64 B): u64 magic "KCBTMODL", u32 version 1, i32 n_tensors, i32 world_size,
 *     i32 grad dtype, i64 step, u64 layout hash, i64 cap_bytes, u32 CRC-32 of every byte
 *     after the header, u32 pad[3];
 *   per tensor i: i64 index, i64 numel, u32 CRC-32 of p, m, v, u32 pad; then p, m, v
 *     (numel fp32 each, the tensor's elements in order; padding is not written).
 * Written to `path`.tmp, fsync'd, renamed.  Host-only; may run while training runs (a half
 * rewritten during the export is CM_ERR_STATE, nothing is left behind).  *step_out (may be
 * NULL) = the step written.  CM_ERR_CONFIG if the table or world size does not match the
 * segments; CM_ERR_STATE if a shard does not hold `step`; CM_ERR_ARG for I/O errors.    */
cm_status cm_shadow_export(const char *shm_name, const cm_layer_table *table, int32_t world_size, int64_t step,
                           const char *path, int64_t *step_out);
const char *cm_last_error(const cm_ctx *ctx);

/* ------------------------------------------------------------------ hot path
 * cm_allreduce_multicast -- reduce-scatter + tap + all-gather of bucket b for iteration
 * t, one fused sm_100a kernel on `stream` (sec 2.1 AllReduce =
 * ReduceScatter + AllGather; sec 4.1.1 "deliver each reduced
 * gradient to the shadow cluster exactly once per iteration").  Rank r owns shard r:
 *   R[i] = (((g_0[i] + g_1[i]) + g_2[i]) + ... + g_{n-1}[i])   fp32, rank order (R2, R3)
 * (bf16 grads: exact upcast, fp32 sum, one round-to-nearest-even to bf16, R14/R25), read
 * from the n ranks' buffers over NVLink; stored once into the host ring slot t mod D
 * (the tap) and into shard r of all n ranks' grad buffers (the all-gather).  In place:
 * only rank r touches shard r of any buffer.  Cross-rank readiness is handled inside the
 * kernel by epoch-tagged flags; the call is stream-ordered after the caller's writes of
 * bucket b.  Before the first bucket of iteration t >= D, the stream waits until the
 * shadow released slot t mod D (lossless backpressure, sec 4.3.3): if
 * the matching cm_shadow_apply was never enqueued the call fails with CM_ERR_STATE
 * instead of overwriting an unconsumed slot.  Iterations are consecutive (CM_ERR_STATE
 * on a gap); buckets of one iteration may be issued in any order, each exactly once.  */
cm_status cm_allreduce_multicast(cm_ctx *ctx, int32_t bucket, int64_t iteration, void *stream);

/* cm_apply_step -- the training replica's AdamW step `step` = t+1 over all P_pad
 * elements, one fused HBM-bound sm_100a kernel (reading R4):
 *   g = R*inv_n; m = B1*m + c1*g; v = B2*v + c2*(g*g); mh = m/bc1; vh = v/bc2;
 *   d = sqrt(vh) + eps; p = p - lr*(mh/d + wd*p)
 * every op an IEEE fp32 op rounded to nearest, no FMA; scalars c1=1-b1, c2=1-b2,
 * bc1=1-b1^s, bc2=1-b2^s, inv_n=1/n computed in fp64 on the host and rounded once (R5,
 * R6).  Requires every bucket of iteration t to have been all-reduced (CM_ERR_STATE
 * otherwise: "no partial update").  Records the step's scalars for the
 * shadow.  With CM_FLAG_NO_TAP the all-reduce has no tap and no shadow exists.        */
cm_status cm_apply_step(cm_ctx *ctx, int64_t step, const cm_adamw *hp, void *stream);

/* cm_apply_step_sgd -- the same step with SGD-momentum instead of AdamW (SPEC.md:310-316,
 * reading R27), one fused HBM-bound kernel over the same flat buffers:
 *   g = R*inv_n; d = g  (or g + wd*p when weight_decay != 0); buf = mu*buf + d;
 *   p = p - lr*buf
 * fp32 IEEE ops, no FMA.  The velocity buf lives in the m buffer; v is not read or
 * written (keep it zero).  The step's optimizer kind and scalars go into the ring-slot
 * record, so the shadow and restore roll-forward replay SGD with identical bits.  The
 * first step of a context fixes its optimizer: switching between cm_apply_step and
 * cm_apply_step_sgd later is CM_ERR_STATE.  Same preconditions and errors as
 * cm_apply_step; works with CM_FLAG_ZERO1 (velocity shard-local).                    */
cm_status cm_apply_step_sgd(cm_ctx *ctx, int64_t step, const cm_sgd *hp, void *stream);

/* cm_apply_bucket -- the training step `step` for ONE bucket, as soon as that bucket's
 * all-reduce is issued ("the backward pass overlaps gradient
 * computation and synchronization"): the optimizer of the bucket's elements runs on
 * `stream` right behind its all-reduce (typically the DDP communication stream), overlapping
 * the rest of the backward pass instead of running after it.  Same element arithmetic and
 * bits as cm_apply_step.  Multi-process ranks: the kernel starts with a per-bucket fence
 * (every rank's all-reduce of the bucket finished).  ZeRO-1: this rank's shard of the
 * bucket, fused with the parameter all-gather.  Every bucket of a step must use identical
 * hyper-parameters; all ranks must call it for the same buckets in the same order (like the
 * all-reduces).  cm_apply_step(step) then finishes the step: it applies the buckets not yet
 * applied and records the step's scalars for the shadow.  CM_ERR_STATE: bucket not
 * all-reduced in this iteration, applied twice, other hyper-parameters; CM_ERR_INVARIANT
 * after a non-finite report.                                                            */
cm_status cm_apply_bucket(cm_ctx *ctx, int32_t bucket, int64_t step, const cm_adamw *hp, void *stream);
cm_status cm_apply_bucket_sgd(cm_ctx *ctx, int32_t bucket, int64_t step, const cm_sgd *hp, void *stream);

/* cm_shadow_apply -- the shadow replica's step `step` (Listing 2, PAPER.md:290-298:
 * "buckets.recv(); optimizer.step()"), enqueued on `side_stream`, off the training
 * stream's critical path.  Waits (stream-ordered) until every tap of iteration step-1 is
 * in the ring ("Once all gradients for an iteration are received"), then
 * applies the identical AdamW to shard r of the shadow state, reading the ring slot and
 * ping-pong half (step-1)&1, writing half step&1, publishes the step in the segment
 * header and releases the ring slot.  step must be last+1 (CM_ERR_STATE: an iteration
 * gap is fatal) and cm_apply_step(step) must have been called.          */
cm_status cm_shadow_apply(cm_ctx *ctx, int64_t step, void *side_stream);

/* cm_restore -- the failure path (PAPER.md:313-314 consolidation; sec 6.5 methodology,
 * PAPER.md:601).  Collective over the n ranks.  Reads every rank's segment header,
 * computes the consolidation step I (reading R21: the largest step every shard can reach
 * -- its published step, its retained previous half, or by rolling forward over fully
 * tapped ring slots), rolls this rank's shard forward to I if needed, copies it host ->
 * device and all-gathers p/m/v to every rank over NVLink.  Blocks until done; returns I
 * in *restored_step; the caller resumes at iteration I.  CM_ERR_UNRECOVERABLE if no
 * common step exists.  Host shadow: a rolled-forward step I is persisted into the half
 * that is NOT the roll-forward source (a half beyond I is invalidated first), so a kill
 * during restore leaves a segment from which the next cm_restore reaches I again.      */
cm_status cm_restore(cm_ctx *ctx, int64_t *restored_step, void *stream);
/* Preconditions and effects of cm_restore, beyond the above:
 *   - every rank calls it after quiescing its own work (no kernel of the context in flight:
 *     synchronise the device) and after a process-group barrier, so every rank reads the
 *     same durable segment headers and computes the same I;
 *   - it is the recovery from CM_ERR_INVARIANT (non-finite): I precedes the flagged step,
 *     and the report is cleared;
 *   - after every rank has computed I (the all-gather's entry barrier), this rank's log above
 *     I is invalidated (ring records, tap flags, snapshot halves): those steps will be
 *     recomputed, possibly with other gradients, and must never be rolled forward.        */

/* ------------------------------------------------------------------ inputs / checks
 * cm_gen_grads -- synthetic gradients (gradient production) for this
 * rank at iteration t into the registered grad buffer, from the counter-based generator
 * of DESIGN.md "Input recipe" (SplitMix64; padding elements are zero).                 */
cm_status cm_gen_grads(cm_ctx *ctx, uint64_t seed, int64_t iteration, int32_t scale, void *stream);
/* cm_init_state -- p = p_0 from the generator (identical on every rank), m = v = 0.    */
cm_status cm_init_state(cm_ctx *ctx, uint64_t seed, void *stream);

/* cm_verify -- bitwise compare this rank's shadow shard (current half) with shard r of
 * the training p, m, v.  Synchronises `stream`.  *mismatch = -1 if
 * equal, else the flat index of the first differing element; CM_ERR_INVARIANT then.
 * Same as cm_verify_ex(ctx, CM_VERIFY_SHADOW, mismatch, NULL, stream).                 */
cm_status cm_verify(cm_ctx *ctx, int64_t *mismatch, void *stream);

/* cm_verify_ex -- the bytes that carry the paper's claim, checked bitwise against the
 * training replica at its current step T ("identical ... to the 8th decimal",
 * reading R18 bitwise).  Synchronises the device.  `scope` is a mask:
 *   CM_VERIFY_SHADOW  the shadow's working state at its published step (must equal T) vs
 *                     shard r of training p/m/v (+ the host snapshot half if it is at T)
 *   CM_VERIFY_HOST    HOST placement: the restore source alone -- the newest host snapshot
 *                     <= T rolled forward over the tapped ring slots with their recorded
 *                     scalars (what cm_restore computes; every step must be recoverable from
 *                     host memory) -- vs training p/m/v; chunked through library scratch
 *   CM_VERIFY_RING    the ring slot of iteration T-1 (host memory, shard-local) vs the reduced
 *                     gradients the training step consumed: shard r of the grad buffer (the
 *                     caller must not have overwritten it since step T), or with ZeRO-1 the
 *                     staging half
 * Results: CM_OK, *mismatch = -1, *what = -1; or CM_ERR_INVARIANT with *mismatch = the
 * smallest differing flat index and *what = 0 p, 1 m, 2 v, 3 ring gradient; *what = 4: a
 * kernel reported a non-finite value (*mismatch = its flat index, -1 unknown); *what = 5:
 * the host log cannot reach step T (a gap).  CM_ERR_STATE if the shadow is not at T.     */
#define CM_VERIFY_SHADOW 1
#define CM_VERIFY_HOST 2
#define CM_VERIFY_RING 4
cm_status cm_verify_ex(cm_ctx *ctx, int32_t scope, int64_t *mismatch, int32_t *what, void *stream);

/* cm_barrier -- a stream-ordered cross-GPU barrier (one tiny kernel; collective: every rank
 * calls it in the same position of its call sequence).  Used to start timed regions of all
 * ranks together (bench.py's lockstep all-reduce chain).  No-op for virtual ranks / n = 1.  */
cm_status cm_barrier(cm_ctx *ctx, void *stream);

/* cm_check -- the non-finite report, without synchronising: CM_ERR_INVARIANT with *step =
 * the first flagged step and *index = a flat element index of it (-1 unknown) once a
 * kernel that already ran saw an inf/NaN; CM_OK with *step = -1 otherwise.  Either pointer
 * may be NULL.  Cleared by cm_restore.                                                    */
cm_status cm_check(cm_ctx *ctx, int64_t *step, int64_t *index);

/* Introspection (host-only, cheap). */
typedef struct {
    int32_t n_buckets, world_size, rank, ring_depth, grad_dtype, shadow_place, peers_in_process;
    int32_t drain_ctas;                 /* how tap drains / snapshot persists reach the host
                                           now: 0 copy engine, k > 0 a k-CTA SM drain kernel
                                           (cm_set_param "drain_ctas": -1 auto, the default) */
    int32_t numa_node;                  /* NUMA node the host segment was placed on, -1 none
                                           (cm_set_param "numa_node")                     */
    int64_t padded_numel, shard_numel;  /* P_pad; sum over buckets of E_b/n               */
    int64_t shadow_step;                /* last step the shadow published                 */
    int64_t launches;                   /* kernels this context launched so far           */
    uint64_t layout_hash;
    int64_t nonfinite_step;             /* first step flagged non-finite, -1 none (cm_verify_ex) */
    int64_t nonfinite_index;            /* a flat element index of that step, -1 unknown       */
    int32_t persist_every;              /* K in effect (host shadows across processes: >= 2)   */
    int32_t pad0;
    int64_t host_half_step[2];          /* step held by each snapshot half (HOST: the host halves;
                                           DEVICE: the HBM halves), -1 invalid              */
} cm_info;
cm_status cm_get_info(const cm_ctx *ctx, cm_info *out);
cm_status cm_bucket_info(const cm_ctx *ctx, int32_t bucket, int64_t *elem_off, int64_t *padded,
                         int64_t *used);
/* Host pointers into the shadow: state half h (0/1) as shard-local arrays of
 * shard_numel fp32 (HOST placement only; DEVICE placement returns device pointers),
 * and ring slot k (shard-local, grad dtype).  For tests and tools.                     */
/* cm_join -- make `stream` wait for everything the library has enqueued on its internal
 * streams so far (copy-engine tap drains to the host ring, shadow staging/persist copies).
 * Stream-ordered, no host synchronisation.  Benchmarks call it before stopping a timer.   */
cm_status cm_join(cm_ctx *ctx, void *stream);

/* cm_set_param -- tuning knobs used by benchmarks and ablations (defaults are the
 * measured best); CM_ERR_ARG for an unknown key or out-of-range value.
 *   "adamw_impl"          AdamW data movement (same arithmetic): 0 per-thread 128-bit items,
 *                         1 TMA bulk-copy staged, 2 warp-tiled 512-byte runs (default; at
 *                         the measured HBM copy bandwidth on B200 vs 82% / 77%), 3 warp-tiled
 *                         one tile per iteration with 4 blocks per SM (ablation)
 *   "adam_blocks"         grid cap of the training AdamW kernel
 *   "tma_blocks"          grid of the TMA AdamW kernel (default: one block per SM)
 *   "ar_blocks"           grid cap of the all-reduce kernel at n >= 2 (default: co-resident
 *                         blocks of the n-rank instance; must be equal on every rank)
 *   "ar_blocks_tap_only"  grid cap of the all-reduce kernel at n == 1, where it is only the
 *                         PCIe-bound tap (default 32: leaves SMs to the shadow and training)
 *   "shadow_blocks"       grid cap of the vectorised shadow AdamW
 * Collective knobs (every rank must set the same value, before the first all-reduce):
 *   "oneshot_max_bytes"   buckets up to this size take the one-shot push kernel (SURVEY 8
 *                         f2; default 2 MiB / n, at most 1 MiB; 0 disables)
 *   "lazy_exit"           1 (default): no exit barrier per bucket, the training step's
 *                         optimizer kernel starts with one iteration fence; 0: an exit
 *                         barrier per bucket (each all-reduce a complete collective)
 *   "force_no_barriers"   profiling only, before cm_connect: in-process ranks on several GPUs run
 *                         without the cross-GPU barriers, so ncu can serialise their kernels
 *                         (the data is then not a valid all-reduce; the NVLink traffic is)
 *   "pdl_mode"            experiments on the PDL trigger (bit 0: no wait for the predecessor
 *                         before exit -- completion order no longer guaranteed; bit 1: trigger
 *                         after the data phase); default 0
 *   "pdl"                 1: launch the all-reduce kernels with programmatic dependent launch
 *                         (multi-process ranks, and n = 1): the next bucket's kernel launches
 *                         and passes its entry barrier while the previous one still moves data
 *                         (n = 1: the staging copies of consecutive buckets overlap their
 *                         launch and ramp; 0.96 vs 0.69 of HBM per GPT-2 bucket).  It waits
 *                         for its stream predecessor only when that was not one of this
 *                         context's all-reduces, so the caller must not write gradients with
 *                         its own kernels on the all-reduce stream between two calls (produce
 *                         them on another stream + event, as a DDP comm stream does).  0
 *                         (default): plain stream order.  Only with lazy exits (an all-reduce
 *                         with an exit barrier is launched in plain stream order); 2 forces
 *                         PDL with exit barriers too (test of the monotone barrier slots)
 *   "ar_grid_switch_bytes" buckets up to this size take one block per SM instead of the
 *                         co-resident cap (default 48 MiB; ignored once "ar_blocks" is set)
 *   "ar_impl"             -1 (default) auto: the bulk-copy pipeline for buckets of at least
 *                         "ar_tma_min_bytes" (default 12 MiB), the unrolled kernel below; 0
 *                         unrolled two-shot kernel (per-thread 16-byte loads/stores), 1
 *                         software-pipelined variant, 2 bulk-copy pipeline (TMA pulls of every
 *                         rank's tile into shared memory, bulk-store pushes; staged tap / no
 *                         tap, n >= 2) for every bucket
 *   "ar_pipe_blocks"      grid of ar_impl 1 (default 148, one block per SM)
 *   "zero1_impl"          ZeRO-1 AdamW + parameter all-gather kernel: 1 (default) two
 *                         4-element groups per thread in flight, 0 one (ablation), 2 the
 *                         updated parameters staged in shared memory per 2048-element tile
 *                         and pushed to every rank's p with cp.async.bulk stores
 * Per-rank knobs:
 *   "drain_ctas"          how tap drains and snapshot persists reach the host: -1 (default)
 *                         auto policy from the GPU-timed step period, 0 copy
 *                         engine, k > 0 a k-CTA SM drain kernel
 *   "numa_node"           NUMA placement of the host shadow segment (set before cm_connect):
 *                         -2 (default) the node of the GPU's PCIe root from sysfs, -1 the
 *                         kernel's first-touch default, k >= 0 node k; MPOL_PREFERRED, best
 *                         effort (cm_info.numa_node reports the outcome)
 *   "shadow_after_train"  1 (default): the shadow step starts after the training step's
 *                         optimizer kernel, so the two HBM-bound optimizer kernels do not
 *                         share the memory system on the step's critical path (GPT-2 model
 *                         mode, n=1: -0.2 ms per step); 0: after the iteration's last all-reduce
 *   "n1_copy_engine"      1: with one rank the staged tap's copy of each bucket into the HBM
 *                         staging half is a copy-engine copy instead of a kernel (ablation)
 *   "persist_queue"       1: snapshot persists go on the tap-drain stream (drains and persists
 *                         take the device->host link one at a time); 0 (default) their own
 *                         low-priority stream
 *   "drain_flush_bytes"   a pending run of adjacent tap drains is issued at this size
 *                         (default 8 MiB, at most 64 MiB)
 *   "ablate_no_drain"     1: staged taps are never drained to the host ring (cost ablation;
 *                         only with CM_FLAG_NO_SHADOW -- restore would be impossible)        */
cm_status cm_set_param(cm_ctx *ctx, const char *key, int64_t value);

/* cm_timing -- per-kernel device timing with CUDA events recorded on each kernel's own
 * stream around its launch (after any stream waits).  enable=1 clears and starts
 * collecting; enable=0 stops, synchronises the events and returns the summed
 * milliseconds and launch counts per class into ms_out[7] / count_out[7] (either may be
 * NULL): 0 all-reduce+tap kernel, 1 training AdamW, 2 shadow AdamW kernel (on its own
 * stream, after its waits), 3 gradient
 * generation, 4 restore copy, 5 tap drains (device->host copies or SM-drain launches of
 * the staged tap, on the drain stream), 6 snapshot persists (device->host, on the persist
 * stream).  Used by bench.py for the roofline of each kernel and the host link's busy
 * time.                                                                                */
cm_status cm_timing(cm_ctx *ctx, int32_t enable, double *ms_out, int64_t *count_out);
/* cm_timing_bytes -- bytes moved device->host by classes 5 (tap drains) and 6 (snapshot
 * persists) in the last closed cm_timing window, per class into bytes_out[7] (other
 * classes 0): the persists that actually fell in the window, not an average.           */
cm_status cm_timing_bytes(const cm_ctx *ctx, int64_t *bytes_out);
cm_status cm_shadow_view(const cm_ctx *ctx, int32_t half, float **p, float **m, float **v);
cm_status cm_ring_view(const cm_ctx *ctx, int32_t slot, void **grads);

#ifdef __cplusplus
}
#endif
#endif /* CM_H_ */
