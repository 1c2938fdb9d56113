/*
 * cm_oracle.c -- the CPU ORACLE for the Checkmate hot path (arXiv 2507.13522).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2507_13522_b200/, libcm.so) never includes, links or calls anything here,
 * and this file includes no header of the product path: the two share no code.
 *
 * Plain, slow, obviously-correct C.  Compiled with -O2 -ffp-contract=off and no
 * fast-math, on x86-64 (SSE scalar float: every float op below is one IEEE binary32
 * operation rounded to nearest-even; no FMA contraction, no extended precision).
 * The precision is binary32 because the method fixes it: the paper's vision models
 * train in fp32 and its LM models in bf16 (sec 6.1), the optimizer
 * state is fp32, and the whole point of the method is that the shadow applies the
 * SAME deterministic fp32 step as the trainer (sec 1
 * sec 3.3).  fp64 appears only where DESIGN.md reading R5/R6 puts it (host scalars).
 *
 * Every function cites the passage it follows.  Readings of silent / ambiguous
 * points are numbered R1..R26 and listed in DESIGN.md section "Readings".
 *
 * Pins: tests/test_oracle_pins.py checks every function here against things other
 * than itself (SPEC worked examples, closed forms, brute force in numpy float32
 * scalars, fp64 error bounds, the public SplitMix64 test vector, torch's bf16 cast).
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <math.h>
#include <xmmintrin.h>
#include <pmmintrin.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CMO_F32 0
#define CMO_BF16 1

/* ------------------------------------------------------------------------- */
/* 0. Environment check: FTZ / DAZ must be off (R17: no flush of subnormals). */
/* ------------------------------------------------------------------------- */
/* threads the sampled trajectory uses (1 unless built with -fopenmp) */
int cmo_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int cmo_fp_env_ok(void) {
    unsigned int csr = _mm_getcsr();
    int ftz = (csr & _MM_FLUSH_ZERO_MASK) != 0;
    int daz = (csr & _MM_DENORMALS_ZERO_MASK) != 0;
    int rn = (csr & _MM_ROUND_MASK) == _MM_ROUND_NEAREST;
    return (!ftz && !daz && rn) ? 1 : 0;
}

/* ------------------------------------------------------------------------- */
/* 1. Bucket planner.                                                        */
/* PAPER.md:258-264 (sec 4.2.2): "group parameters by bin-packing them,       */
/* starting from the last model layer and working backwards to the first.    */
/* A model layer is mapped to a bucket until the bucket size is less than the */
/* maximum given size, such as 25MB ... If a layer size exceeds the bucket    */
/* size, it is mapped to a single dedicated bucket."                          */
/* Reading R10: add while bucket bytes <= cap; a tensor */
/* larger than cap gets its own bucket, closing the current one.  R13: the    */
/* unit is a parameter tensor.  R12/R26: each bucket is padded   */
/* with zeros to a multiple of n*V elements, V = 16 bytes / elem_size, so it  */
/* splits into n equal 16-byte-aligned shards.                                */
/* Flat layout: bucket 0 first; inside a bucket, tensors in the order added   */
/* (i.e. reverse model order); padding at the end of each bucket.             */
/* Outputs: bucket_first[b] = first tensor index added to b (the highest      */
/* index), bucket_count[b] = number of tensors, bucket_off[b] = flat element  */
/* offset, bucket_padded[b] = padded element count, bucket_used[b] = real    */
/* (unpadded) element count, tensor_off[i] = flat element offset of tensor i. */
/* Returns the bucket count, or -1 on bad input (sizes > 0).     */
/* ------------------------------------------------------------------------- */
int64_t cmo_plan(const int64_t *numel, int32_t n_tensors, int64_t cap_bytes,
                 int32_t elem_size, int32_t world_size,
                 int32_t *bucket_first, int32_t *bucket_count,
                 int64_t *bucket_off, int64_t *bucket_padded, int64_t *bucket_used,
                 int64_t *tensor_off, int64_t *total_padded) {
    if (n_tensors <= 0 || cap_bytes <= 0 || world_size <= 0) return -1;
    if (elem_size != 4 && elem_size != 2) return -1;
    for (int32_t i = 0; i < n_tensors; ++i) if (numel[i] <= 0) return -1;
    int64_t quantum = (16 / elem_size) * (int64_t)world_size;
    /* pass 1: group tensors, walking backwards from the last one */
    int64_t nb = 0, cur_bytes = 0;
    for (int32_t i = n_tensors - 1; i >= 0; --i) {
        int64_t bytes = numel[i] * elem_size;
        int open = nb > 0 && bucket_count[nb - 1] > 0 && cur_bytes >= 0;
        if (bytes > cap_bytes) {                    /* dedicated bucket, closes the open one */
            bucket_first[nb] = i; bucket_count[nb] = 1; nb++;
            cur_bytes = -1;                          /* -1: no open bucket */
            continue;
        }
        if (open && cur_bytes + bytes <= cap_bytes) {   /* still fits: add */
            bucket_count[nb - 1]++;
            cur_bytes += bytes;
        } else {                                     /* start a new bucket */
            bucket_first[nb] = i; bucket_count[nb] = 1; nb++;
            cur_bytes = bytes;
        }
    }
    /* pass 2: flat offsets; tensors inside bucket b are first, first-1, ... */
    int64_t flat = 0;
    for (int64_t b = 0; b < nb; ++b) {
        int64_t used = 0;
        bucket_off[b] = flat;
        for (int32_t k = 0; k < bucket_count[b]; ++k) {
            int32_t i = bucket_first[b] - k;
            tensor_off[i] = flat + used;
            used += numel[i];
        }
        bucket_used[b] = used;
        bucket_padded[b] = ((used + quantum - 1) / quantum) * quantum;
        flat += bucket_padded[b];
    }
    *total_padded = flat;
    return nb;
}

/* ------------------------------------------------------------------------- */
/* 2. Synthetic inputs.  A counter-based generator */
/* so any element of any rank at any iteration can be regenerated alone.      */
/* This is not the method's arithmetic; the product implements the same       */
/* generator independently (the two share no code).                           */
/* SplitMix64 finaliser (Steele, Lea, Flood, OOPSLA 2014; public reference    */
/* splitmix64.c): sm(x) = mix(x + 0x9E3779B97F4A7C15).                         */
/* ------------------------------------------------------------------------- */
uint64_t cmo_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t cmo_hash(uint64_t seed, uint64_t r, uint64_t t, uint64_t i) {
    return cmo_splitmix64(cmo_splitmix64(seed ^ (r << 48) ^ t) ^ i);
}

/* fp32 gradient: mantissa int24 in [-2^23, 2^23), scale 2^(-23-e-s), e in 0..7.
 * Exactly representable in binary32 (<= 24 significant bits, power-of-two scale). */
float cmo_gen_f32(uint64_t seed, uint64_t r, uint64_t t, uint64_t i, int32_t s) {
    uint64_t h = cmo_hash(seed, r, t, i);
    int32_t e = (int32_t)((h >> 32) & 7u);
    int32_t mant = (int32_t)(h >> 40) - (1 << 23);
    return ldexpf((float)mant, -23 - e - s);
}

/* bf16 gradient: mantissa int8 in [-128, 128), scale 2^(-7-e-s); returned as
 * the binary32 value (exactly representable in bf16, so the bf16 bits are the
 * top 16 bits of the float). */
float cmo_gen_bf16val(uint64_t seed, uint64_t r, uint64_t t, uint64_t i, int32_t s) {
    uint64_t h = cmo_hash(seed, r, t, i);
    int32_t e = (int32_t)((h >> 32) & 7u);
    int32_t mant = (int32_t)(h >> 56) - 128;
    return ldexpf((float)mant, -7 - e - s);
}

static uint16_t f32_hi16(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); }
static float bf16_to_f32(uint16_t b) { uint32_t u = ((uint32_t)b) << 16; float f; memcpy(&f, &u, 4); return f; }

/* Initial master weight p_0[i] (identical on every rank: DP replicas start equal,
 * PAPER.md:62 sec 2.1).  R19: the shadow starts from this same state
 * ("applies them to a prior checkpoint replica"). */
float cmo_gen_p0(uint64_t seed, uint64_t i) {
    return ldexpf(cmo_gen_f32(seed, 0xFFFF, 0, i, 0), -5);
}

/* Fill the flat padded gradient buffer of rank r at iteration t.  Padding
 * elements (R26) are zero.  `out` is float* for F32, uint16_t* for BF16. */
void cmo_fill_grads(uint64_t seed, int32_t r, int64_t t, int32_t dtype, int32_t s,
                    int64_t n_buckets, const int64_t *bucket_off, const int64_t *bucket_padded,
                    const int64_t *bucket_used, void *out) {
    for (int64_t b = 0; b < n_buckets; ++b) {
        for (int64_t k = 0; k < bucket_padded[b]; ++k) {
            int64_t i = bucket_off[b] + k;
            int used = k < bucket_used[b];
            if (dtype == CMO_F32) {
                ((float *)out)[i] = used ? cmo_gen_f32(seed, (uint64_t)r, (uint64_t)t, (uint64_t)i, s) : 0.0f;
            } else {
                ((uint16_t *)out)[i] = used ? f32_hi16(cmo_gen_bf16val(seed, (uint64_t)r, (uint64_t)t, (uint64_t)i, s)) : 0;
            }
        }
    }
}

void cmo_fill_p0(uint64_t seed, int64_t n_buckets, const int64_t *bucket_off,
                 const int64_t *bucket_padded, const int64_t *bucket_used, float *p) {
    for (int64_t b = 0; b < n_buckets; ++b)
        for (int64_t k = 0; k < bucket_padded[b]; ++k) {
            int64_t i = bucket_off[b] + k;
            p[i] = k < bucket_used[b] ? cmo_gen_p0(seed, (uint64_t)i) : 0.0f;
        }
}

/* ------------------------------------------------------------------------- */
/* 3. Reduce (the value an all-reduce delivers).                              */
/* PAPER.md:67-69 (sec 2.1): "During ReduceScatter, each node splits its      */
/* gradients into chunks, exchanges these chunks with other nodes, and reduces*/
/* them (e.g., by summing ...)."  R1: the wire carries the SUM (1/n is the    */
/* optimizer's first op).  R2: fixed rank order 0,1,...,n-1 for every element */
/* (north_star "fixed rank-order reduction").  R3: the accumulator is seeded  */
/* with g_0 (not +0.0), so -0 + -0 stays -0.                                  */
/* R[i] = fl(...fl(fl(g_0[i] + g_1[i]) + g_2[i]) ... + g_{n-1}[i]).           */
/* ------------------------------------------------------------------------- */
void cmo_reduce_f32(int32_t n, int64_t len, const float *const *g, float *R) {
    for (int64_t i = 0; i < len; ++i) {
        float acc = g[0][i];
        for (int32_t k = 1; k < n; ++k) acc = acc + g[k][i];
        R[i] = acc;
    }
}

/* R25: binary32 -> bf16 round-to-nearest-even on the bit pattern (finite inputs). */
uint16_t cmo_f32_to_bf16_rne(float f) {
    uint32_t u; memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

/* R14: bf16 grads are upcast exactly, summed in fp32 in rank order, then
 * rounded ONCE to bf16 (the value both the all-gather and the tap carry). */
void cmo_reduce_bf16(int32_t n, int64_t len, const uint16_t *const *g, uint16_t *R) {
    for (int64_t i = 0; i < len; ++i) {
        float acc = bf16_to_f32(g[0][i]);
        for (int32_t k = 1; k < n; ++k) acc = acc + bf16_to_f32(g[k][i]);
        R[i] = cmo_f32_to_bf16_rne(acc);
    }
}

/* ------------------------------------------------------------------------- */
/* 4. AdamW step scalars (host side, once per step).                          */
/* AdamW as SPEC.md:318-326 ([OP] adamw_step; the paper cites AdamW only,     */
/* PAPER.md:307 sec 4.2.4, sec 6.1).  R5: each scalar computed in */
/* fp64 then rounded once to fp32.  R6: beta^s by s repeated fp64 multiplies   */
/* starting from 1.0 (no pow).  R7: s = t+1 >= 1.                              */
/* out[0..9] = { c1=1-b1, c2=1-b2, B1=b1, B2=b2, bc1=1-b1^s, bc2=1-b2^s,        */
/*               inv_n=1/n, lr, eps, wd }                                      */
/* ------------------------------------------------------------------------- */
int cmo_scalars(int64_t s, double lr, double beta1, double beta2, double eps,
                double wd, int32_t n, float *out) {
    if (s < 1 || n < 1) return -1;
    double p1 = 1.0, p2 = 1.0;
    for (int64_t k = 0; k < s; ++k) { p1 = p1 * beta1; p2 = p2 * beta2; }
    out[0] = (float)(1.0 - beta1);
    out[1] = (float)(1.0 - beta2);
    out[2] = (float)beta1;
    out[3] = (float)beta2;
    out[4] = (float)(1.0 - p1);
    out[5] = (float)(1.0 - p2);
    out[6] = (float)(1.0 / (double)n);
    out[7] = (float)lr;
    out[8] = (float)eps;
    out[9] = (float)wd;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* 5. AdamW element update, canonical fp32 op sequence (R4):      */
/*   g  = R * inv_n                                                            */
/*   m  = B1*m + c1*g                                                          */
/*   v  = B2*v + c2*(g*g)                                                      */
/*   mh = m / bc1 ;  vh = v / bc2                                              */
/*   d  = sqrt(vh) + eps                                                       */
/*   p  = p - lr*(mh/d + wd*p)          (p on the right is the old p)          */
/* Each operation rounded to nearest, no FMA (north_star: "fp32 IEEE ops       */
/* without FMA contraction in the optimizer").                                 */
/* ------------------------------------------------------------------------- */
static void adamw_elem(float R, const float *sc, float *p, float *m, float *v) {
    float c1 = sc[0], c2 = sc[1], B1 = sc[2], B2 = sc[3], bc1 = sc[4], bc2 = sc[5];
    float inv_n = sc[6], lr = sc[7], eps = sc[8], wd = sc[9];
    float g = R * inv_n;
    float mm = B1 * (*m) + c1 * g;
    float gg = g * g;
    float vv = B2 * (*v) + c2 * gg;
    float mh = mm / bc1;
    float vh = vv / bc2;
    float d = sqrtf(vh) + eps;
    float upd = mh / d + wd * (*p);
    float pp = (*p) - lr * upd;
    *m = mm; *v = vv; *p = pp;
}

void cmo_adamw_f32(int64_t len, const float *R, const float *sc, float *p, float *m, float *v) {
    for (int64_t i = 0; i < len; ++i) adamw_elem(R[i], sc, &p[i], &m[i], &v[i]);
}

void cmo_adamw_bf16(int64_t len, const uint16_t *R, const float *sc, float *p, float *m, float *v) {
    for (int64_t i = 0; i < len; ++i) adamw_elem(bf16_to_f32(R[i]), sc, &p[i], &m[i], &v[i]);
}

/* ------------------------------------------------------------------------- */
/* 6. One full data-parallel iteration of the path, whole-buffer form, and    */
/* the shadow.  PAPER.md:274-275 (Listing 1: backward = gradient sync, then    */
/* optimizer.step()); PAPER.md:290-298 (Listing 2: shadow buckets.recv();     */
/* optimizer.step()).  The tap T_t equals R_t exactly and once (*/
/* "deliver each reduced gradient to the shadow cluster exactly once per      */
/* iteration").  The shadow applies the same step to its own copy (PAPER.md:32,*/
/* 154: "Once all gradients for an iteration are received, shadow nodes run   */
/* the optimizer step").                                                       */
/* grads: n pointers to per-rank flat buffers (float* or uint16_t*); R, T:    */
/* outputs (same dtype), train/shadow p,m,v: in/out, total elements.          */
/* ------------------------------------------------------------------------- */
void cmo_iteration(int32_t n, int64_t total, int32_t dtype, const void *const *grads,
                   const float *sc, void *R, void *T,
                   float *tp, float *tm, float *tv, float *sp, float *sm, float *sv) {
    if (dtype == CMO_F32) {
        cmo_reduce_f32(n, total, (const float *const *)grads, (float *)R);
        memcpy(T, R, (size_t)total * 4);                 /* tap: exactly R, once */
        cmo_adamw_f32(total, (const float *)R, sc, tp, tm, tv);
        if (sp) cmo_adamw_f32(total, (const float *)T, sc, sp, sm, sv);
    } else {
        cmo_reduce_bf16(n, total, (const uint16_t *const *)grads, (uint16_t *)R);
        memcpy(T, R, (size_t)total * 2);
        cmo_adamw_bf16(total, (const uint16_t *)R, sc, tp, tm, tv);
        if (sp) cmo_adamw_bf16(total, (const uint16_t *)T, sc, sp, sm, sv);
    }
}

/* ------------------------------------------------------------------------- */
/* 7. Sampled trajectories (C2/C4 at full size).  The step is elementwise      */
/* independent -- the paper's "functional optimizer" property*/
/* ("the optimizer step for each parameter is deterministic and independent   */
/* of the others") -- so element i's state after `steps` iterations depends    */
/* only on p_0[i] and g_{r,t}[i], which the counter-based generator yields     */
/* without materialising anything else.  idx[] are flat padded indices;        */
/* used[] says whether the index is a real parameter (else padding: g=p0=0).   */
/* Outputs p,m,v after `steps` steps and R of the last iteration (as float;    */
/* for bf16 the bf16-rounded value).  Scalars use lr etc. constant over steps. */
/* ------------------------------------------------------------------------- */
/* initial state of the sampled elements: p = p_0 (padding 0), m = v = 0 */
void cmo_sample_init(uint64_t seed, int64_t n_idx, const int64_t *idx, const uint8_t *used,
                     float *p, float *m, float *v, float *R_last) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n_idx; ++k) {
        p[k] = used[k] ? cmo_gen_p0(seed, (uint64_t)idx[k]) : 0.0f;
        m[k] = 0.0f; v[k] = 0.0f; R_last[k] = 0.0f;
    }
}

/* iterations t0 .. t0+steps-1 of the sampled elements' trajectories (state in/out) */
void cmo_sample_iterate(uint64_t seed, int32_t n, int32_t dtype, int32_t gscale,
                        int64_t t0, int64_t steps, double lr, double b1, double b2,
                        double eps, double wd, int64_t n_idx, const int64_t *idx,
                        const uint8_t *used, float *p, float *m, float *v, float *R_last) {
    float sc[10];
    for (int64_t t = t0; t < t0 + steps; ++t) {
        cmo_scalars(t + 1, lr, b1, b2, eps, wd, n, sc);
        /* elements are independent: the all-core timing build
           (-fopenmp, bench.py's cpu_baseline) splits them over threads; the same
           per-element arithmetic, and without -fopenmp the pragma is ignored */
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < n_idx; ++k) {
            uint64_t i = (uint64_t)idx[k];
            float R;
            if (dtype == CMO_F32) {
                float acc = used[k] ? cmo_gen_f32(seed, 0, (uint64_t)t, i, gscale) : 0.0f;
                for (int32_t r = 1; r < n; ++r)
                    acc = acc + (used[k] ? cmo_gen_f32(seed, (uint64_t)r, (uint64_t)t, i, gscale) : 0.0f);
                R = acc;
            } else {
                float acc = used[k] ? cmo_gen_bf16val(seed, 0, (uint64_t)t, i, gscale) : 0.0f;
                for (int32_t r = 1; r < n; ++r)
                    acc = acc + (used[k] ? cmo_gen_bf16val(seed, (uint64_t)r, (uint64_t)t, i, gscale) : 0.0f);
                R = bf16_to_f32(cmo_f32_to_bf16_rne(acc));
            }
            adamw_elem(R, sc, &p[k], &m[k], &v[k]);
            R_last[k] = R;
        }
    }
}

void cmo_run_sample(uint64_t seed, int32_t n, int32_t dtype, int32_t gscale,
                    int64_t t0, int64_t steps, double lr, double b1, double b2,
                    double eps, double wd, int64_t n_idx, const int64_t *idx,
                    const uint8_t *used, float *p, float *m, float *v, float *R_last) {
    cmo_sample_init(seed, n_idx, idx, used, p, m, v, R_last);
    cmo_sample_iterate(seed, n, dtype, gscale, t0, steps, lr, b1, b2, eps, wd, n_idx, idx, used,
                       p, m, v, R_last);
}

/* ------------------------------------------------------------------------- */
/* 7b. SGD with momentum.  PAPER.md:307 (sec 4.2.4) names SGD*/
/* among the functional optimizers the shadow can replay     */
/* ([OP] sgd_step) fixes the update: velocity' = momentum*velocity + g,        */
/* p' = p - lr*velocity' (momentum = 0 gives p' = p - lr*g).                   */
/* Reading R27: g = R * inv_n first (R1, as for AdamW); when       */
/* weight_decay != 0 the coupled L2 term of the classic SGD form is added to   */
/* the gradient, d = g + wd*p (old p), a host-side choice recorded as wd_on;   */
/* with wd = 0 the SPEC form is used unchanged.  The velocity is stored in the */
/* m array (v is unused).  Scalars: fp64 -> fp32 once (R5).                    */
/* out[0..4] = { mu, inv_n, lr, wd, wd_on (1.0f or 0.0f) }                      */
/* ------------------------------------------------------------------------- */
int cmo_sgd_scalars(double lr, double momentum, double wd, int32_t n, float *out) {
    if (n < 1) return -1;
    out[0] = (float)momentum;
    out[1] = (float)(1.0 / (double)n);
    out[2] = (float)lr;
    out[3] = (float)wd;
    out[4] = wd != 0.0 ? 1.0f : 0.0f;
    return 0;
}

/*   g   = R * inv_n                                                           */
/*   d   = g            (wd_on = 0)   |   d = g + wd*p   (wd_on = 1)            */
/*   buf = mu*buf + d                                                          */
/*   p   = p - lr*buf                                                          */
static void sgd_elem(float R, const float *sc, float *p, float *buf) {
    float mu = sc[0], inv_n = sc[1], lr = sc[2], wd = sc[3];
    float g = R * inv_n;
    float d = g;
    if (sc[4] != 0.0f) d = g + wd * (*p);
    float b = mu * (*buf) + d;
    float pp = (*p) - lr * b;
    *buf = b; *p = pp;
}

void cmo_sgd_f32(int64_t len, const float *R, const float *sc, float *p, float *buf) {
    for (int64_t i = 0; i < len; ++i) sgd_elem(R[i], sc, &p[i], &buf[i]);
}

void cmo_sgd_bf16(int64_t len, const uint16_t *R, const float *sc, float *p, float *buf) {
    for (int64_t i = 0; i < len; ++i) sgd_elem(bf16_to_f32(R[i]), sc, &p[i], &buf[i]);
}

/* Sampled SGD trajectory (same element independence as cmo_run_sample,       */
/* PAPER.md:306-308).  Outputs p and the velocity buf after `steps` steps.     */
void cmo_run_sample_sgd(uint64_t seed, int32_t n, int32_t dtype, int32_t gscale,
                        int64_t t0, int64_t steps, double lr, double momentum, double wd,
                        int64_t n_idx, const int64_t *idx, const uint8_t *used,
                        float *p, float *buf, float *R_last) {
    float sc[5];
    cmo_sgd_scalars(lr, momentum, wd, n, sc);
    for (int64_t k = 0; k < n_idx; ++k) {
        p[k] = used[k] ? cmo_gen_p0(seed, (uint64_t)idx[k]) : 0.0f;
        buf[k] = 0.0f; R_last[k] = 0.0f;
    }
    for (int64_t t = t0; t < t0 + steps; ++t) {
        for (int64_t k = 0; k < n_idx; ++k) {
            uint64_t i = (uint64_t)idx[k];
            float R;
            if (dtype == CMO_F32) {
                float acc = used[k] ? cmo_gen_f32(seed, 0, (uint64_t)t, i, gscale) : 0.0f;
                for (int32_t r = 1; r < n; ++r)
                    acc = acc + (used[k] ? cmo_gen_f32(seed, (uint64_t)r, (uint64_t)t, i, gscale) : 0.0f);
                R = acc;
            } else {
                float acc = used[k] ? cmo_gen_bf16val(seed, 0, (uint64_t)t, i, gscale) : 0.0f;
                for (int32_t r = 1; r < n; ++r)
                    acc = acc + (used[k] ? cmo_gen_bf16val(seed, (uint64_t)r, (uint64_t)t, i, gscale) : 0.0f);
                R = bf16_to_f32(cmo_f32_to_bf16_rne(acc));
            }
            sgd_elem(R, sc, &p[k], &buf[k]);
            R_last[k] = R;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* 8. Consolidation target for restore.  PAPER.md:313-314 ("uses a           */
/* configurable timeout to consolidate shards into a complete checkpoint");   */
/* R21 / SPEC.md:413-421: I = min over shards of the last completed step.     */
/* ------------------------------------------------------------------------- */
int64_t cmo_consolidate(int32_t n_shards, const int64_t *last_step) {
    int64_t I = last_step[0];
    for (int32_t r = 1; r < n_shards; ++r) if (last_step[r] < I) I = last_step[r];
    return I;
}
