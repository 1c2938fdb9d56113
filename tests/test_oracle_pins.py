"""Pins for the CPU oracle (oracle/cm_oracle.c): each test checks the oracle against
something other than itself -- SPEC worked examples, closed forms, brute force in numpy
float32 scalars, fp64 error bounds, public test vectors, torch's library routines.
CPU only (no GPU marker)."""
import math
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2507_13522_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold_lines(name):
    with open(os.path.join(GOLD, name)) as f:
        return [l.strip() for l in f if l.strip() and not l.startswith("#")]


def f32bits(x):
    return int(np.array([x], np.float32).view(np.uint32)[0])


def test_fp_environment():
    assert O.lib().cmo_fp_env_ok() == 1  # R17: no FTZ/DAZ, round-to-nearest


# ----------------------------------------------------------------------------- generator
def test_splitmix64_public_vector():
    golden = 0x9E3779B97F4A7C15
    for line in _gold_lines("splitmix64.txt"):
        k, val = line.split()
        assert O.lib().cmo_splitmix64((int(k) * golden) % 2**64) == int(val, 16)


def _np_hash(seed, r, t, i):
    """Independent numpy re-derivation of the counter hash (uint64 wraparound)."""
    M = np.uint64

    def sm(x):
        z = (x + M(0x9E3779B97F4A7C15))
        z = (z ^ (z >> M(30))) * M(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> M(27))) * M(0x94D049BB133111EB)
        return z ^ (z >> M(31))
    with np.errstate(over="ignore"):
        return sm(sm(M(seed) ^ (M(r) << M(48)) ^ M(t)) ^ i.astype(np.uint64))


@pytest.mark.parametrize("s", [0, 10, 12])
def test_generator_exact_and_distributed(s):
    idx = np.arange(0, 1 << 14, dtype=np.int64) * 7919
    vals = np.array([O.lib().cmo_gen_f32(3, 1, 5, int(i), s) for i in idx], np.float64)
    h = _np_hash(3, 1, 5, idx)
    e = ((h >> np.uint64(32)) & np.uint64(7)).astype(np.int64)
    mant = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    expect = mant.astype(np.float64) * np.exp2(-23.0 - e - s)
    np.testing.assert_array_equal(vals, expect)                 # exact, no rounding
    assert np.all(np.float32(vals) == vals)                      # representable in fp32
    assert abs(vals.mean()) < 4 * vals.std() / math.sqrt(len(vals))
    assert set(np.unique(e)) == set(range(8))                    # 8 binades of spread
    bf = np.array([O.lib().cmo_gen_bf16val(3, 1, 5, int(i), s) for i in idx[:2048]], np.float32)
    assert np.all((bf.view(np.uint32) & 0xFFFF) == 0)            # exactly representable in bf16
    mant8 = (h[:2048] >> np.uint64(56)).astype(np.int64) - 128
    np.testing.assert_array_equal(bf.astype(np.float64), mant8 * np.exp2(-7.0 - e[:2048] - s))


def test_generator_padding_is_zero_and_p0_small():
    plan = O.Plan(W.numels(W.c1_ragged()), 1 << 20, 4, 8)
    g = O.gen_grads(plan, 0, 1, 2, O.F32)
    p = O.gen_p0(plan, 0)
    used = plan.used_mask().astype(bool)
    assert np.all(g[~used] == 0) and np.all(p[~used] == 0)
    assert np.count_nonzero(g[used]) > 0.99 * used.sum()
    assert np.abs(p).max() < 2.0 ** -5


# ----------------------------------------------------------------------------- planner
def test_planner_spec_examples():
    for line in _gold_lines("planner_spec_examples.txt"):
        sizes, cap, exp = [x.strip() for x in line.split("|")]
        sizes = [int(x) for x in sizes.split(",")]
        # sizes are bytes; use 2-byte elements so numel = bytes / 2
        plan = O.Plan([s // 2 for s in sizes], int(cap), 2, 1)
        groups = []
        for b in range(plan.n_buckets):
            groups.append([plan.bucket_first[b] - k for k in range(plan.bucket_count[b])])
        expect = [[int(x) for x in g.split(",")] for g in exp.split(";")]
        assert groups == expect, (line, groups)


def test_planner_rejects_bad_tables():
    for bad in ([], [0], [5, -1]):
        with pytest.raises(ValueError):
            O.Plan(bad, 100, 4, 1)


def _check_plan_properties(numel, cap, es, n):
    plan = O.Plan(numel, cap, es, n)
    q = (16 // es) * n
    seen = []
    flat = 0
    for b in range(plan.n_buckets):
        ts = [plan.bucket_first[b] - k for k in range(plan.bucket_count[b])]
        seen += ts
        assert plan.bucket_off[b] == flat
        assert plan.bucket_padded[b] % q == 0 and plan.bucket_padded[b] >= plan.bucket_used[b]
        assert plan.bucket_padded[b] - plan.bucket_used[b] < q
        assert (plan.bucket_off[b] * es) % 16 == 0 and (plan.bucket_padded[b] // n * es) % 16 == 0
        nbytes = sum(numel[i] for i in ts) * es
        if len(ts) > 1:
            assert nbytes <= cap
        else:
            assert nbytes <= cap or numel[ts[0]] * es > cap
        o = flat
        for i in ts:
            assert plan.tensor_off[i] == o
            o += numel[i]
        assert plan.bucket_used[b] == o - flat
        # greedy maximality: the next tensor (if any) did not fit or was oversized
        nxt = ts[-1] - 1
        if nxt >= 0 and numel[ts[0]] * es <= cap:
            assert nbytes + numel[nxt] * es > cap
        flat += plan.bucket_padded[b]
    assert seen == list(range(len(numel) - 1, -1, -1))       # every tensor once, reverse order
    assert plan.total == flat
    return plan


def test_planner_properties_random():
    rng = np.random.default_rng(0)
    for _ in range(300):
        nt = int(rng.integers(1, 40))
        numel = [int(x) for x in rng.integers(1, 5000, nt)]
        cap = int(rng.integers(4, 40000))
        es = int(rng.choice([2, 4]))
        n = int(rng.choice([1, 2, 3, 4, 8]))
        _check_plan_properties(numel, cap, es, n)


def test_planner_paper_models():
    # GPT-2 small, fp32 grads, 25 MiB: 16 buckets + 1 dedicated wte bucket
    p = _check_plan_properties(W.numels(W.gpt2_small()), W.CAP_BYTES, 4, 8)
    assert p.n_buckets == 17 and p.total == 124439808
    assert p.bucket_count[-1] == 1 and p.bucket_first[-1] == 0        # wte last, dedicated
    p = _check_plan_properties(W.numels(W.llama3_8b()), W.CAP_BYTES, 2, 8)
    assert p.n_buckets == 226 and p.total == 8030261248
    p = _check_plan_properties(W.numels(W.c1()), 1 << 20, 4, 2)
    assert p.n_buckets == 4 and list(p.bucket_padded) == [262144] * 4


# ----------------------------------------------------------------------------- reduce
def _numpy_rank_order(gs):
    acc = gs[0].astype(np.float32).copy()
    for g in gs[1:]:
        acc = (acc + g.astype(np.float32)).astype(np.float32)   # numpy float32 add, IEEE RN
    return acc


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_reduce_brute_force_tiny(n):
    rng = np.random.default_rng(n)
    specials = np.array([0.0, -0.0, 1e-45, -1e-45, 1.17549435e-38, 2.0**24, -(2.0**24), 1.0, 3.0e38],
                        np.float32)
    for trial in range(50):
        L = int(rng.integers(1, 64))
        gs = []
        for k in range(n):
            g = (rng.standard_normal(L) * np.exp2(rng.integers(-30, 30, L))).astype(np.float32)
            mask = rng.random(L) < 0.2
            g[mask] = rng.choice(specials[:-1], mask.sum())
            gs.append(g)
        R = O.reduce_f32(gs)
        ref = _numpy_rank_order(gs)
        np.testing.assert_array_equal(R.view(np.uint32), ref.view(np.uint32))


def test_reduce_order_and_signed_zero():
    # R2: [1, 2^24, -2^24] is 0 in rank order, 1 in ring-cyclic order starting at rank 1
    gs = [np.array([1.0], np.float32), np.array([2.0**24], np.float32), np.array([-(2.0**24)], np.float32)]
    assert O.reduce_f32(gs)[0] == 0.0
    assert O.reduce_f32([gs[1], gs[2], gs[0]])[0] == 1.0
    # R3: seeded with g_0, so -0 + -0 = -0 (a +0.0 seed would give +0)
    z = [np.array([-0.0], np.float32)] * 4
    assert f32bits(O.reduce_f32(z)[0]) == 0x80000000


def test_reduce_integer_values_exact_vs_fp64():
    rng = np.random.default_rng(7)
    for n in (2, 4, 8):
        gs = [rng.integers(-(1 << 20), 1 << 20, 4096).astype(np.float32) for _ in range(n)]
        exact = np.sum(np.stack(gs).astype(np.float64), axis=0)
        np.testing.assert_array_equal(O.reduce_f32(gs).astype(np.float64), exact)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_reduce_fp64_error_bound(n):
    # north_star: within 1e-6 relative of an fp64 reference sum; reading R15: |R - S64| <= 1e-6 * sum|g|
    plan = O.Plan(W.numels(W.c1()), 1 << 20, 4, n)
    gs = [O.gen_grads(plan, 0, r, 0, O.F32) for r in range(n)]
    R = O.reduce_f32(gs).astype(np.float64)
    G = np.stack(gs).astype(np.float64)
    S = G.sum(0)
    A = np.abs(G).sum(0)
    gamma = (n - 1) * 2.0 ** -24 / (1 - (n - 1) * 2.0 ** -24)   # Higham's gamma_{n-1}
    assert np.all(np.abs(R - S) <= gamma * A)
    assert np.all(np.abs(R - S) <= 1e-6 * A)


def test_reduce_n2_commutative_equals_any_order():
    # with two summands fp32 + is commutative, so any all-reduce order gives these bits
    rng = np.random.default_rng(1)
    a = rng.standard_normal(10000).astype(np.float32)
    b = rng.standard_normal(10000).astype(np.float32)
    np.testing.assert_array_equal(O.reduce_f32([a, b]), O.reduce_f32([b, a]))
    np.testing.assert_array_equal(O.reduce_f32([a, b]), (torch.from_numpy(a) + torch.from_numpy(b)).numpy())


def test_bf16_rne_matches_torch_cast():
    rng = np.random.default_rng(2)
    x = (rng.standard_normal(200000) * np.exp2(rng.integers(-40, 40, 200000))).astype(np.float32)
    # add exact ties: low 16 bits = 0x8000 with both parities of bit 16
    ties = (rng.integers(0x00800000, 0x7F000000, 4000).astype(np.uint32) & 0xFFFF0000) | 0x8000
    x = np.concatenate([x, ties.view(np.float32), -ties.view(np.float32)])
    ours = np.array([O.f32_to_bf16(v) for v in x[:20000]] +
                    [O.f32_to_bf16(v) for v in x[-8000:]], np.uint16)
    ref = torch.from_numpy(np.concatenate([x[:20000], x[-8000:]])).to(torch.bfloat16).view(torch.int16).numpy()
    np.testing.assert_array_equal(ours, ref.view(np.uint16))


def test_reduce_bf16_is_rne_of_fp32_rank_sum():
    plan = O.Plan(W.numels(W.c1()), 1 << 20, 2, 4)
    gs = [O.gen_grads(plan, 0, r, 3, O.BF16)[:50000] for r in range(4)]
    up = [(g.astype(np.uint32) << 16).view(np.float32) for g in gs]
    ref32 = _numpy_rank_order(up)
    ref = torch.from_numpy(ref32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(O.reduce_bf16(gs), ref)


# ----------------------------------------------------------------------------- scalars
def test_scalar_bits():
    gold = dict(l.rsplit(None, 1) for l in _gold_lines("fp32_scalar_bits.txt"))
    sc = O.scalars(1, b1=0.9, b2=0.999).view(np.uint32)
    assert sc[0] == int(gold["fl32(1-0.9)"], 16) and sc[1] == int(gold["fl32(1-0.999)"], 16)
    naive1 = np.float32(1.0) - np.float32(0.9)
    naive2 = np.float32(1.0) - np.float32(0.999)
    assert f32bits(naive1) == int(gold["1.0f-0.9f"], 16) and f32bits(naive2) == int(gold["1.0f-0.999f"], 16)
    # s = 1: bias corrections equal c1, c2 (1 - beta^1)
    assert sc[4] == sc[0] and sc[5] == sc[1]


def test_scalar_bias_correction_vs_libm_pow():
    # R6: repeated multiplication; fl32(1 - beta^s) agrees with libm pow for these betas
    for b in (0.9, 0.95, 0.98, 0.999):
        for s in list(range(1, 200)) + [1000, 5000, 20000]:
            sc = O.scalars(s, b1=b, b2=b)
            assert sc[4] == np.float32(1.0 - math.pow(b, s)), (b, s)
    assert O.scalars(10 ** 5, b1=0.9, b2=0.999)[4] == np.float32(1.0)
    for n in (1, 2, 4, 8):
        assert O.scalars(1, n=n)[6] == np.float32(1.0 / n)
    with pytest.raises(ValueError):
        O.scalars(0)


# ----------------------------------------------------------------------------- AdamW
def test_adamw_spec_example():
    d = dict(l.split() for l in _gold_lines("adamw_spec_example.txt"))
    sc = O.scalars(int(d["step"]), lr=float(d["lr"]), wd=float(d["wd"]))
    p = np.array([0], np.uint32).view(np.float32).copy()
    m = np.zeros(1, np.float32)
    v = np.zeros(1, np.float32)
    O.adamw(np.array([int(d["g"], 16)], np.uint32).view(np.float32), sc, p, m, v)
    assert f32bits(p[0]) == int(d["p1"], 16)


@pytest.mark.parametrize("n", [1, 2, 8])
def test_adamw_first_step_power_of_two_closed_form(n):
    # s=1, m=v=0, R = n*g with g = +-2^k: m_hat = g, v_hat = g^2, d = |g| (eps below half-ulp
    # for |g| >= 2^-2), so p' = p - lr*(+-1 + wd*p) exactly.
    rng = np.random.default_rng(n)
    for k in range(-2, 8):
        for sgn in (1.0, -1.0):
            p0 = rng.standard_normal(64).astype(np.float32)
            p, m, v = p0.copy(), np.zeros(64, np.float32), np.zeros(64, np.float32)
            sc = O.scalars(1, lr=1e-3, wd=0.01, n=n)
            O.adamw(np.full(64, sgn * n * 2.0 ** k, np.float32), sc, p, m, v)
            lr, wd = np.float32(1e-3), np.float32(0.01)
            expect = p0 - lr * (np.float32(sgn) + wd * p0)
            np.testing.assert_array_equal(p, expect.astype(np.float32))
            np.testing.assert_array_equal(m, (sc[0] * np.float32(sgn * 2.0 ** k)).astype(np.float32))


def test_adamw_fixed_point_and_pure_decay():
    p0 = np.random.default_rng(0).standard_normal(1000).astype(np.float32)
    p, m, v = p0.copy(), np.zeros(1000, np.float32), np.zeros(1000, np.float32)
    O.adamw(np.zeros(1000, np.float32), O.scalars(3, wd=0.0), p, m, v)
    np.testing.assert_array_equal(p, p0)                     # g=0, m=v=0, wd=0: fixed point
    assert np.all(m == 0) and np.all(v == 0)
    O.adamw(np.zeros(1000, np.float32), O.scalars(4, lr=1e-2, wd=0.1), p, m, v)
    # 0/(0+eps) = 0, so only decoupled decay acts: p - lr*(0 + wd*p)
    np.testing.assert_array_equal(p, (p0 - np.float32(1e-2) * (np.float32(0) + np.float32(0.1) * p0)))


def test_adamw_multistep_vs_torch_fp64():
    """Sanity vs textbook AdamW (torch.optim.AdamW in float64): tolerance only."""
    rng = np.random.default_rng(5)
    N = 5000
    p0 = (rng.standard_normal(N) * 0.05).astype(np.float32)
    grads = [(rng.standard_normal(N) * np.exp2(rng.integers(-12, 0, N))).astype(np.float32) for _ in range(20)]
    p, m, v = p0.copy(), np.zeros(N, np.float32), np.zeros(N, np.float32)
    tp = torch.nn.Parameter(torch.from_numpy(p0.astype(np.float64)))
    opt = torch.optim.AdamW([tp], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, foreach=False)
    for s, g in enumerate(grads, start=1):
        O.adamw(g, O.scalars(s), p, m, v)
        tp.grad = torch.from_numpy(g.astype(np.float64))
        opt.step()
    ref = tp.detach().numpy()
    assert np.max(np.abs(p - ref)) < 1e-6, np.max(np.abs(p - ref))
    st = opt.state[tp]
    em, ev = st["exp_avg"].numpy(), st["exp_avg_sq"].numpy()
    # fp32 vs fp64 rounding, relative to the running scale (m cancels, so not plain relative)
    np.testing.assert_allclose(m, em, rtol=1e-5, atol=1e-5 * np.abs(em).max())
    np.testing.assert_allclose(v, ev, rtol=1e-5, atol=1e-5 * np.abs(ev).max())
    # the update moved p (a dropped term or wrong sign would fail the tolerance above)
    assert np.max(np.abs(p - p0)) > 1e-3


def test_adamw_partition_invariance():
    # PAPER.md:306-308 "functional optimizer": any shard split gives identical bytes
    rng = np.random.default_rng(3)
    N = 10007
    R = rng.standard_normal(N).astype(np.float32)
    p0 = rng.standard_normal(N).astype(np.float32)
    whole = [p0.copy(), np.zeros(N, np.float32), np.zeros(N, np.float32)]
    sc = O.scalars(2)
    O.adamw(R, sc, *whole)
    for k in (2, 3, 7):
        parts = [p0.copy(), np.zeros(N, np.float32), np.zeros(N, np.float32)]
        cuts = np.linspace(0, N, k + 1).astype(int)
        for a, b in zip(cuts[:-1], cuts[1:]):
            sub = [x[a:b].copy() for x in parts]
            O.adamw(R[a:b].copy(), sc, *sub)
            for x, y in zip(parts, sub):
                x[a:b] = y
        for x, y in zip(parts, whole):
            np.testing.assert_array_equal(x.view(np.uint32), y.view(np.uint32))


# ----------------------------------------------------------------------------- run / shadow / restore
def test_run_tap_equals_reduce_and_shadow_equals_train():
    plan = O.Plan(W.numels(W.c1_ragged()), 1 << 20, 4, 2)
    run = O.Run(plan, seed=1)
    for _ in range(3):
        gs = run.step()
        np.testing.assert_array_equal(run.T, run.R)                       # tap carries R exactly once
        np.testing.assert_array_equal(run.R, O.reduce_f32(gs))
        for a, b in ((run.p, run.sp), (run.m, run.sm), (run.v, run.sv)):
            np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
    used = plan.used_mask().astype(bool)
    assert np.all(run.p[~used] == 0) and np.all(run.m[~used] == 0)       # padding stays 0


@pytest.mark.parametrize("dtype", [O.F32, O.BF16])
def test_run_sample_matches_whole_buffer(dtype):
    es = 4 if dtype == O.F32 else 2
    plan = O.Plan(W.numels(W.c1_ragged()), 1 << 20, es, 4)
    run = O.Run(plan, seed=2, dtype=dtype)
    for _ in range(4):
        run.step()
    idx = np.random.default_rng(0).choice(plan.total, 3000, replace=False).astype(np.int64)
    used = plan.used_mask()[idx]
    p, m, v, R = O.run_sample(2, 4, dtype, 10, 4, idx, used)
    np.testing.assert_array_equal(p, run.p[idx])
    np.testing.assert_array_equal(m, run.m[idx])
    np.testing.assert_array_equal(v, run.v[idx])
    Rw = run.R[idx] if dtype == O.F32 else (run.R[idx].astype(np.uint32) << 16).view(np.float32)
    np.testing.assert_array_equal(R, Rw)


def test_restore_continues_bit_exact_and_consolidation_rule():
    plan = O.Plan(W.numels(W.c1()), 1 << 20, 4, 2)
    ctl = O.Run(plan, seed=4, shadow=False)
    for _ in range(6):
        ctl.step()
    a = O.Run(plan, seed=4)
    for _ in range(3):
        a.step()
    # "fail" at k=3: restore from the shadow state (sec 6.5) and continue
    b = O.Run(plan, seed=4, shadow=False)
    b.p, b.m, b.v, b.t = a.sp.copy(), a.sm.copy(), a.sv.copy(), 3
    for _ in range(3):
        b.step()
    for x, y in ((b.p, ctl.p), (b.m, ctl.m), (b.v, ctl.v)):
        np.testing.assert_array_equal(x.view(np.uint32), y.view(np.uint32))
    # SPEC.md:419-421 consolidation examples
    assert O.consolidate([10, 10]) == 10
    assert O.consolidate([10, 9]) == 9
    assert O.consolidate([7, 9, 8, 7]) == 7


# ----------------------------------------------------------------------------- SGD-momentum (f4)
def test_sgd_spec_examples():
    for line in _gold_lines("sgd_spec_examples.txt"):
        p0, g, lr, mu, p1 = line.split()
        p = np.array([int(p0, 16)], np.uint32).view(np.float32).copy()
        buf = np.zeros(1, np.float32)
        O.sgd(np.array([int(g, 16)], np.uint32).view(np.float32), O.sgd_scalars(lr=float(lr), momentum=float(mu)),
              p, buf)
        assert f32bits(p[0]) == int(p1, 16)


@pytest.mark.parametrize("n", [1, 2, 8])
def test_sgd_geometric_momentum_closed_form(n):
    # mu = 1/2, constant g = 2^k, lr = 2^-10, wd = 0, buf_0 = 0: buf_t = g (2 - 2^(1-t)) and
    # p_t = p_0 - lr g (2t - 2 + 2^(1-t)); every intermediate has few significant bits, so
    # both are exact in binary32.  R = n*g checks that inv_n is applied first.
    for k in (-3, 0, 4):
        g = 2.0 ** k
        p = np.full(4, 1.0, np.float32)
        buf = np.zeros(4, np.float32)
        sc = O.sgd_scalars(lr=2.0 ** -10, momentum=0.5, wd=0.0, n=n)
        for t in range(1, 13):
            O.sgd(np.full(4, n * g, np.float32), sc, p, buf)
            assert np.all(buf == np.float32(g * (2.0 - 2.0 ** (1 - t)))), (k, t)
            assert np.all(p == np.float32(1.0 - 2.0 ** -10 * g * (2 * t - 2 + 2.0 ** (1 - t)))), (k, t)


def test_sgd_pure_weight_decay_closed_form():
    # g = 0, mu = 0, wd = 1/2, lr = 1/2: d = p/2, buf = d, p' = p - p/4 = (3/4) p,
    # so p_t = (3/4)^t exactly while 3^t < 2^24 (t <= 15)
    p = np.ones(3, np.float32)
    buf = np.zeros(3, np.float32)
    sc = O.sgd_scalars(lr=0.5, momentum=0.0, wd=0.5)
    for t in range(1, 16):
        O.sgd(np.zeros(3, np.float32), sc, p, buf)
        assert np.all(p == np.float32(0.75 ** t)), t
    # zero gradient without decay is a fixed point
    q = np.random.default_rng(0).standard_normal(100).astype(np.float32)
    q0, b = q.copy(), np.zeros(100, np.float32)
    O.sgd(np.zeros(100, np.float32), O.sgd_scalars(lr=0.1, momentum=0.9), q, b)
    np.testing.assert_array_equal(q, q0)


def test_sgd_multistep_vs_torch_fp64():
    """Sanity vs torch.optim.SGD (momentum, coupled weight decay) in float64: tolerance only."""
    rng = np.random.default_rng(6)
    N = 5000
    p0 = (rng.standard_normal(N) * 0.05).astype(np.float32)
    grads = [(rng.standard_normal(N) * np.exp2(rng.integers(-12, 0, N))).astype(np.float32) for _ in range(20)]
    p, buf = p0.copy(), np.zeros(N, np.float32)
    tp = torch.nn.Parameter(torch.from_numpy(p0.astype(np.float64)))
    opt = torch.optim.SGD([tp], lr=1e-2, momentum=0.9, weight_decay=1e-4, foreach=False)
    sc = O.sgd_scalars(lr=1e-2, momentum=0.9, wd=1e-4)
    for g in grads:
        O.sgd(g, sc, p, buf)
        tp.grad = torch.from_numpy(g.astype(np.float64))
        opt.step()
    ref = tp.detach().numpy()
    assert np.max(np.abs(p - ref)) < 1e-6, np.max(np.abs(p - ref))
    eb = opt.state[tp]["momentum_buffer"].numpy()
    np.testing.assert_allclose(buf, eb, rtol=1e-5, atol=1e-5 * np.abs(eb).max())
    assert np.max(np.abs(p - p0)) > 1e-3


@pytest.mark.parametrize("dtype", [O.F32, O.BF16])
def test_sgd_run_sample_matches_whole_buffer_and_shadow(dtype):
    es = 4 if dtype == O.F32 else 2
    plan = O.Plan(W.numels(W.c1_ragged()), 1 << 20, es, 2)
    hp = dict(lr=1e-2, momentum=0.9, wd=1e-4)
    run = O.Run(plan, seed=3, dtype=dtype, opt="sgd", hp=hp)
    for _ in range(4):
        run.step()
        for a, b in ((run.p, run.sp), (run.m, run.sm)):
            np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
        assert not run.v.any() and not run.sv.any()
    idx = np.random.default_rng(1).choice(plan.total, 3000, replace=False).astype(np.int64)
    used = plan.used_mask()[idx]
    p, b, R = O.run_sample_sgd(3, 2, dtype, 10, 4, idx, used, **hp)
    np.testing.assert_array_equal(p, run.p[idx])
    np.testing.assert_array_equal(b, run.m[idx])
