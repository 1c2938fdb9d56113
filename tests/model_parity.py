"""Model-mode parity from GradProbe records: with real backward gradients the
inputs cannot be regenerated, so every rank keeps, at sampled flat indices, its gradients
before the reduce and the state before the step; the oracle then recomputes the rank-order
reduce (bitwise, and within 1e-6 * sum|g| of the fp64 sum, reading R15) and the AdamW step of
those elements (bitwise) and compares them with every rank's post-step values.
Test infrastructure: imports the oracle."""
import numpy as np

from oracle import oracle as O


def probe_indices(ddp, k, seed=0):
    """k random used flat indices plus every bucket's first and last used element."""
    r = ddp.r
    used = np.zeros(r.padded, bool)
    for off, numel in zip(r.tensor_off, r.numel):
        used[off:off + numel] = True
    cand = np.flatnonzero(used)
    rng = np.random.default_rng(seed)
    idx = rng.choice(cand, min(k, len(cand)), replace=False)
    edges = []
    for off, padded, u in r.buckets():
        edges += [off, off + u - 1]
    return np.unique(np.concatenate([idx, np.asarray(edges, np.int64)])).astype(np.int64)


def check_records(per_rank, n, hp):
    """per_rank[r] = GradProbe.records of rank r (same iterations, same indices)."""
    iters = len(per_rank[0])
    for i in range(iters):
        recs = [pr[i] for pr in per_rank]
        step = recs[0]["step"]
        g = [rec["grad"].numpy().astype(np.float32) for rec in recs]
        R = O.reduce_f32(g)
        S64 = np.sum(np.stack(g).astype(np.float64), axis=0)
        A64 = np.sum(np.abs(np.stack(g).astype(np.float64)), axis=0)
        assert np.all(np.abs(R.astype(np.float64) - S64) <= 1e-6 * A64), f"step {step}: fp64 bound"
        p = recs[0]["p"].numpy().copy()
        m = recs[0]["m"].numpy().copy()
        v = recs[0]["v"].numpy().copy()
        for rec in recs[1:]:                   # replicated state: identical on every rank
            np.testing.assert_array_equal(rec["p"].numpy().view(np.uint32), p.view(np.uint32))
        O.adamw(R, O.scalars(step, lr=hp["lr"], b1=hp["beta1"], b2=hp["beta2"], eps=hp["eps"],
                             wd=hp["weight_decay"], n=n), p, m, v)
        for k, rec in enumerate(recs):
            np.testing.assert_array_equal(rec["R"].numpy().view(np.uint32), R.view(np.uint32),
                                          err_msg=f"R rank {k} step {step}")
            for nm, ref in (("p_new", p), ("m_new", m), ("v_new", v)):
                np.testing.assert_array_equal(rec[nm].numpy().view(np.uint32), ref.view(np.uint32),
                                              err_msg=f"{nm} rank {k} step {step}")
    return {"iterations": iters, "elements": int(len(per_rank[0][0]["R"])) if iters else 0}
