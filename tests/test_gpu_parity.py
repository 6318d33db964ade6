"""Parity of the CUDA path (called through the C-ABI) against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): integer outputs bit-exact; f64 outputs within 1e-6 relative (they are
ratios of exact integers evaluated in the same order, so equality is expected and also asserted).
"""
import dataclasses

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import Params  # noqa: E402

INT_KEYS = ("demand", "batch", "knee", "status", "alloc_q16", "level", "runs", "served", "scen_status", "T_us",
            "misses", "below")
F_KEYS = ("u_static", "u", "thr", "u_ideal", "thr_ideal")


@pytest.fixture(scope="module")
def ds():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_13541_b200 import dstack
    return dstack


def run_gpu(ds, pb, p):
    dp = ds.from_host(pb, "cuda")
    o = ds.eval_batch(dp, p)
    torch.cuda.synchronize()
    return ds.to_numpy(o, pb.num_scen, pb.num_dnn), o


def assert_parity(g, want, keys_f=F_KEYS, ideal=True, where=""):
    for k in INT_KEYS:
        a, b = g[k], want[k]
        if not np.array_equal(a.astype(np.int64), b.astype(np.int64)):
            bad = np.flatnonzero(a.astype(np.int64) != b.astype(np.int64))
            raise AssertionError(f"{where} {k}: {bad.size} mismatches, first at {bad[:8]}: gpu {a[bad[:8]]} oracle {b[bad[:8]]}")
    for k in keys_f:
        if not ideal and k in ("u_ideal", "thr_ideal"):
            continue
        a, b = g[k], want[k]
        np.testing.assert_allclose(a, b, rtol=1e-6, atol=0, err_msg=f"{where} {k}")
        assert np.array_equal(a, b), f"{where} {k}: not bit-identical (max diff {np.max(np.abs(a - b))})"


def test_device_generator_matches_host(ds):
    sp, _ = synth.config(3, num_scen=3000)
    h = synth.generate_host(sp)
    g = synth.generate_device(sp, "cuda")
    torch.cuda.synchronize()
    R = h.num_rows
    for k in ("scen_dnn_off", "dnn_row_off", "t_p", "t_np", "mem_bw", "slo_us", "asm_us", "bmax", "shape"):
        assert np.array_equal(g[k].cpu().numpy(), getattr(h, k)), k
    assert np.array_equal(g["n"][:R].cpu().numpy().view(np.uint32), h.n[:R])
    assert np.array_equal(g["r"][:R].cpu().numpy().view(np.uint16), h.r[:R])
    assert np.array_equal(g["d"][:R].cpu().numpy().view(np.uint32), h.d[:R])


def test_config1_full_parity(ds):
    sp, p = synth.config(1)
    pb = synth.generate_host(sp)
    g, _ = run_gpu(ds, pb, p)
    assert_parity(g, oracle.evaluate(pb, p), where="config1")


VARIANTS = {
    "defaults": dict(),
    "mem_off": dict(mem_mode=0),
    "verbatim": dict(mem_mode=2),
    "per_launch": dict(wse_mode=1),
    "margin": dict(margin=7),
    "bmin": dict(b_min=2, b_max=9),
    "L_eq_S": dict(L=148),
    "L_lt_S_small": dict(L=37),
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_config2_small_parity(ds, name):
    sp, p = synth.config(2, num_scen=120, rows_pct=25)
    p = p.replace(**VARIANTS[name])
    pb = synth.generate_host(sp)
    g, _ = run_gpu(ds, pb, p)
    assert_parity(g, oracle.evaluate(pb, p), where=name)


def test_config2_batching_variant_parity(ds):
    sp, p = synth.config(2, num_scen=80, rows_pct=25, variant="batching")
    pb = synth.generate_host(sp)
    g, _ = run_gpu(ds, pb, p)
    want = oracle.evaluate(pb, p)
    assert_parity(g, want, where="batching")
    assert (want["batch"][want["status"] == 0] > 1).any()   # the variant really exercises b* > 1


def test_knee_curve_parity(ds):
    sp, p = synth.config(2, num_scen=60, rows_pct=30)
    pb = synth.generate_host(sp)
    dp = ds.from_host(pb, "cuda")
    for pp in (p, p.replace(mem_mode=2), p.replace(par_mode=1), p.replace(L=148, wse_mode=1)):
        pbx = pb if pp.par_mode == 0 else synth.generate_host(sp.replace(threads=1))
        dpx = dp if pp.par_mode == 0 else ds.from_host(pbx, "cuda")
        for b in (1, 2, 5, 16, 64):
            k, st = ds.knee(dpx, pp, b)
            ko, sto = oracle.knee(pbx, pp, b)
            assert np.array_equal(st.cpu().numpy(), sto), (b, pp)
            assert np.array_equal(k.cpu().numpy().view(np.uint16), ko), (b, pp)


def test_wmaxmin_parity(ds):
    rng = np.random.default_rng(0)
    sizes = rng.integers(0, 33, 500)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    for L in (1, 50, 100, 148, 255):
        dem = rng.integers(0, L + 3, int(off[-1])).astype(np.uint16)
        dem[rng.random(dem.shape) < 0.1] = 0
        a = ds.wmaxmin(torch.from_numpy(off).cuda(), L, torch.from_numpy(dem.view(np.int16)).cuda())
        a = a.cpu().numpy().view(np.uint32)
        for s in range(len(sizes)):
            want = oracle.wmaxmin(dem[off[s]:off[s + 1]], L)
            assert np.array_equal(a[off[s]:off[s + 1]], want), (L, s)


def test_table4_hook_cycle(ds, golden):
    """Table 4 through dstack_schedule_cycle's test hook: ST-only 59.5%, D-STACK 71.5%."""
    t = golden("table4.json")["models"]
    for names, want_u in ((["Alexnet", "ResNet-50", "VGG-19"], 0.715),
                          (["Alexnet", "Mobilenet", "ResNet-50", "VGG-19"], 0.875)):
        nd = len(names)
        pb = synth.make_problem([0, nd], np.arange(nd + 1), [1] * nd, [1] * nd, [1] * nd,
                                [t[m]["slo_ms"] * 1000 for m in names], [0] * nd, [64] * nd, [1] * nd, [1] * nd,
                                [0] * nd)
        dp = ds.from_host(pb, "cuda")
        p = Params(L=100, S_tot=100, slot_us=100)
        hook = dict(level=torch.tensor([t[m]["knee"] for m in names], dtype=torch.int32, device="cuda"),
                    d_slots=torch.tensor([t[m]["runtime_ms"] * 10 for m in names], dtype=torch.int32, device="cuda"))
        one = torch.ones(nd, dtype=torch.uint8, device="cuda")
        o = ds.schedule_cycle(dp, p, None, one, None, hook=hook)
        torch.cuda.synchronize()
        assert o["misses"][0].item() == 0
        static = sum(int(100000 // (t[m]["slo_ms"] * 1000)) * t[m]["runtime_ms"] * t[m]["knee"] for m in names) / 10000
        assert o["u_static"][0].item() == pytest.approx(static, abs=1e-15)
        assert o["u"][0].item() == pytest.approx(want_u, abs=1e-12)


def test_hook_sessions_random_parity(ds):
    """The a5 session engine alone (dstack_schedule_cycle's test hook: level g_j and run length d_j given, fill at b*
    only) against O5 (oracle.cycle_direct) on random sessions that reach every branch of k_cycle: 1-32 DNNs, L from
    1 to 255, sessions up to 4096 slots, runs inside the 128-slot register window, longer than it (shared-memory
    scans), longer than the session (misses), d >= 8191 (the EDF key's clamp), d = 0."""
    rng = np.random.default_rng(20261017)
    S = 600
    sizes = rng.integers(1, 33, S)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    D = int(off[-1])
    L_of = rng.choice([1, 50, 100, 148, 255], S)
    g = np.zeros(D, np.int32); d = np.zeros(D, np.int32); sl = np.zeros(D, np.int32)
    for s_ in range(S):
        k0, k1 = off[s_], off[s_ + 1]
        T = int(rng.choice([40, 250, 1000, 1024, 1500, 4096]))
        n = k1 - k0
        sl[k0:k1] = np.maximum(1, T // rng.integers(1, 5, n))
        sl[k0 + rng.integers(0, n)] = T                     # the session length
        g[k0:k1] = rng.integers(1, L_of[s_] + 1, n)
        kind = rng.integers(0, 10, n)
        d[k0:k1] = np.where(kind < 5, rng.integers(1, 61, n), np.where(kind < 7, rng.integers(61, 125, n),
                   np.where(kind < 9, rng.integers(125, 700, n), rng.integers(8191, 9001, n))))
        d[k0 + rng.integers(0, n)] = rng.choice([0, 1, 3]) if rng.random() < 0.2 else d[k0]
    one = np.ones(D, np.int32)
    pb = synth.make_problem(off, np.arange(D + 1), one, one, one, sl * 100, np.zeros(D, np.int32), one * 64, one,
                            one, np.zeros(D, np.int32))
    dp = ds.from_host(pb, "cuda")
    o_all = {}
    for Lv in np.unique(L_of):
        p = Params(L=int(Lv), S_tot=148, slot_us=100)
        hook = dict(level=torch.from_numpy(g).cuda(), d_slots=torch.from_numpy(d).cuda())
        o = ds.schedule_cycle(dp, p, None, torch.ones(D, dtype=torch.uint8, device="cuda"), None, hook=hook)
        torch.cuda.synchronize()
        o_all[int(Lv)] = {k: v.cpu().numpy() for k, v in o.items() if v is not None}
    checked = 0
    for s_ in range(S):
        k0, k1 = off[s_], off[s_ + 1]
        o = o_all[int(L_of[s_])]
        nslots = int(sl[k0:k1].max())
        njobs = int(sum(nslots // x for x in sl[k0:k1]))
        if njobs > 512:
            assert o["scen_status"][s_] == 3   # DSTACK_ST_INVALID (capacity, R19)
            continue
        dt = np.zeros((k1 - k0, 64), np.int64); dt[:, 0] = d[k0:k1]
        want = oracle.cycle_direct(g[k0:k1], sl[k0:k1], np.ones(k1 - k0, np.int32), dt, 1, int(L_of[s_]), nslots)
        where = (s_, int(L_of[s_]), nslots)
        assert o["misses"][s_] == want["misses"], where
        assert np.array_equal(o["runs"][k0:k1].view(np.uint16), want["runs"]), where
        assert np.array_equal(o["served"][k0:k1].view(np.uint32), want["served"]), where
        assert o["u_static"][s_] == want["u_static"] and o["u"][s_] == want["u"], where
        checked += 1
    assert checked > S // 2


def test_o8_toys_gpu(ds, golden):
    from tests.test_oracle_sched import toy_problem
    for name in ("A", "B", "C"):
        pb, p, toy = toy_problem(golden, name)
        g, _ = run_gpu(ds, pb, p)
        for k in ("demand", "batch", "alloc_q16", "level", "runs"):
            assert g[k].astype(np.int64).tolist() == toy[k], (name, k)
        assert g["u"][0] == pytest.approx(toy["u"], abs=1e-12)
        assert g["u_ideal"][0] == pytest.approx(toy["u_ideal"], abs=5e-7)
        assert_parity(g, oracle.evaluate(pb, p), where=name)


def edge_problem():
    """Hand-made edge cases: empty scenario, single DNN, invalid / infeasible / overflow DNNs, >32 DNNs,
    a session longer than DSTACK_MAX_SLOTS, SLO not a multiple of the slot, zero-width kernels."""
    from tests.helpers import multi_dnn_problem
    base = dict(rows=[(10, 1, 1000), (3, 2, 500), (0, 1, 0)], t_p=20, t_np=5, M=50000, slo=20000, a=300, bmax=64)
    dnns, sizes = [], []
    sizes.append(0)                                             # empty scenario
    dnns += [base]; sizes.append(1)                             # single DNN
    dnns += [dict(base, t_p=0), dict(base, slo=20050), base]; sizes.append(3)          # invalid members
    dnns += [dict(base, slo=100, a=5000), base]; sizes.append(2)                       # infeasible member
    dnns += [dict(base, rows=[(4_000_000_000, 65535, 4_000_000_000)] * 2, t_p=2**30), base]; sizes.append(2)  # overflow
    dnns += [base] * 33; sizes.append(33)                        # too many DNNs
    dnns += [dict(base, slo=500_000)]; sizes.append(1)           # 5000 slots > DSTACK_MAX_SLOTS
    dnns += [dict(base, rows=[(0, 1, 0)], t_np=0)]; sizes.append(1)                  # latency identically 0
    dnns += [dict(base, rows=[(0, 3, 0), (0, 1, 10)], t_np=1)]; sizes.append(1)      # only zero-width kernels
    dnns += [dict(base, slo=30000), dict(base, slo=100000, rows=[(200, 1, 10**6)] * 40)]; sizes.append(2)  # ragged windows
    return multi_dnn_problem(dnns, sizes)


def test_edge_cases_parity(ds):
    pb = edge_problem()
    for p in (Params(L=100, S_tot=148, ideal=1), Params(L=148, S_tot=148, mem_mode=2, ideal=1)):
        g, _ = run_gpu(ds, pb, p)
        want = oracle.evaluate(pb, p)
        assert_parity(g, want, where="edge")
    assert want["scen_status"].tolist()[:1] == [oracle.INFEASIBLE]
    assert oracle.INVALID in want["status"].tolist() and oracle.OVERFLOW in want["status"].tolist()
    assert oracle.INVALID in want["scen_status"].tolist()


def random_profile_problem(seed, S=260, S_tot=148):
    """Adversarial random DNN profiles for the a1-a3 kernels (fast path, its exactness bands and the generic path):
    1-400 rows of widths from 0 to far beyond S_tot, R up to 3 (and whole DNNs whose R sum reaches 2^16), memory
    bytes from 0 to 2^31, t_np = 0 (ties, the certificate's blind spot) or small, t_p, M, SLO, a and MaxBatch across
    their ranges; 1-6 DNNs per scenario."""
    rng = np.random.default_rng(seed)
    sizes = rng.integers(1, 7, S)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    D = int(off[-1])
    K = rng.integers(1, 401, D)
    K[rng.random(D) < 0.05] = 1
    roff = np.concatenate([[0], np.cumsum(K)]).astype(np.int64)
    R = int(roff[-1])
    kind = rng.choice(4, R, p=[0.3, 0.4, 0.297, 0.003])
    n = np.where(kind == 0, rng.integers(0, 16, R), np.where(kind == 1, rng.integers(1, S_tot + 1, R),
                 np.where(kind == 2, rng.integers(S_tot, 4 * S_tot, R), rng.integers(1, 1 << 16, R)))).astype(np.uint32)
    r = rng.integers(1, 4, R).astype(np.uint16)
    dk = rng.random(R)
    d = np.where(dk < 0.1, 0, np.where(dk < 0.8, rng.integers(0, 10 ** 6, R), np.where(
        dk < 0.97, rng.integers(0, 10 ** 8, R), rng.integers(0, 1 << 31, R, dtype=np.int64)))).astype(np.uint32)
    big = rng.random(D) < 0.03                        # R sums >= 2^16: outside the fast path
    for k in np.flatnonzero(big):
        r[roff[k]:roff[k + 1]] = min(65535, 65535 // max(1, int(K[k])) + 200)
    t_p = rng.integers(1, 41, D).astype(np.int32)
    t_np = np.where(rng.random(D) < 0.25, 0, rng.integers(1, 21, D)).astype(np.int32)
    mbw = rng.integers(1000, 1 << 20, D).astype(np.int32)
    slo = (rng.integers(20, 2001, D) * 100).astype(np.int32)
    asm = rng.integers(0, 3000, D).astype(np.int32)
    bmax = rng.integers(1, 65, D).astype(np.int32)
    return synth.make_problem(off, roff, t_p, t_np, mbw, slo, asm, bmax, n, r, d)


@pytest.mark.parametrize("mode", ["default", "mem_off", "verbatim", "per_launch", "b_min3", "threads", "ideal",
                                  "L_eq_S"])
def test_random_profiles_parity(ds, mode):
    """Whole path (a1-a6 + a8, eval path) on adversarial random profiles vs the oracle: every integer output
    bit-exact, f64 bit-identical."""
    seeds = {"default": 1, "mem_off": 2, "verbatim": 3, "per_launch": 4, "b_min3": 5, "threads": 6, "ideal": 7,
             "L_eq_S": 8}
    pb = random_profile_problem(seeds[mode], S=120 if mode == "ideal" else 260)
    p = Params(L=100, S_tot=148, ideal=0)
    p = {"default": p, "mem_off": p.replace(mem_mode=0), "verbatim": p.replace(mem_mode=2),
         "per_launch": p.replace(wse_mode=1), "b_min3": p.replace(b_min=3), "threads": p.replace(par_mode=1),
         "ideal": p.replace(ideal=1), "L_eq_S": p.replace(L=148)}[mode]
    g, _ = run_gpu(ds, pb, p)
    want = oracle.evaluate(pb, p, nthreads=8)
    assert_parity(g, want, ideal=(mode == "ideal"), where=mode)
    st = want["status"]
    assert (st == 0).sum() > 50   # most DNNs are schedulable, the rest exercise the statuses


def test_ideal_parity_config2(ds):
    sp, p = synth.config(2, num_scen=40, rows_pct=20)
    pb = synth.generate_host(sp)
    g, _ = run_gpu(ds, pb, p)
    assert_parity(g, oracle.evaluate(pb, p), where="ideal")


def test_config3_fullsize_sampled_parity(ds):
    """BASELINE config 3 at full size (1M scenarios) in the launch configuration bench.py times,
    checked on a stratified sample (every 5000th scenario) the oracle computes one by one."""
    sp, p = synth.config(3)
    g = synth.generate_device(sp, "cuda")
    dp = ds.from_device_dict(g)
    o = ds.eval_batch(dp, p)
    torch.cuda.synchronize()
    idx = np.arange(0, sp.num_scen, 5000)
    for s in idx:
        pb = synth.generate_host(sp.replace(scen_base=int(s), num_scen=1))
        want = oracle.evaluate(pb, p)
        k0, k1 = int(g["scen_dnn_off"][s].item()), int(g["scen_dnn_off"][s + 1].item())
        sub = {}
        for k, v in o.items():
            if k == "agg":
                continue
            if k in ("demand", "batch", "knee", "status", "alloc_q16", "level", "runs", "served"):
                a = v[k0:k1].cpu().numpy()
            else:
                a = v[s:s + 1].cpu().numpy()
            sub[k] = a.view(np.uint16) if a.dtype == np.int16 else (a.view(np.uint32) if a.dtype == np.int32 else a)
        assert_parity(sub, want, ideal=False, where=f"cfg3 scen {s}")
    agg = ds.agg_to_dict(o["agg"])
    assert agg["n_scen"] == sp.num_scen and agg["n_dnn"] == dp.num_dnn
    assert sum(agg["n_st"]) == dp.num_dnn and sum(agg["n_scen_st"]) == sp.num_scen


@pytest.mark.parametrize("variant", ["defaults", "verbatim148", "per_launch", "batching"])
def test_split_path_parity(ds, variant):
    """The call-by-call path dstack_batch_opt -> dstack_wmaxmin -> dstack_schedule_cycle (separate kernels)
    against the oracle; dstack_eval_batch uses the fused kernel instead, so both are covered."""
    sp, p = synth.config(2, num_scen=150, rows_pct=25, variant="batching" if variant == "batching" else "default")
    if variant == "verbatim148":
        p = p.replace(mem_mode=2, L=148)
    elif variant == "per_launch":
        p = p.replace(wse_mode=1)
    pb = synth.generate_host(sp)
    dp = ds.from_host(pb, "cuda")
    o = ds.alloc_outputs(dp, agg=False)
    ws = ds.Workspace(ds.workspace_size(dp, p), dp.device)
    ds.batch_opt(dp, p, out=o)
    ds.wmaxmin(dp.scen_dnn_off, p.L, o["demand"], out=o["alloc_q16"])
    ds.schedule_cycle(dp, p, o["demand"], o["batch"], o["alloc_q16"], out=o, ws=ws)
    torch.cuda.synchronize()
    assert_parity(ds.to_numpy(o, pb.num_scen, pb.num_dnn), oracle.evaluate(pb, p), where=f"split-{variant}")


def test_simulate_parity_and_shard_invariance(ds):
    """a7 (config 5) through dstack_simulate vs the oracle's O7; two shards reproduce the single run."""
    sp, p = synth.config(5, num_scen=160, rows_pct=30)
    pb = synth.generate_host(sp)
    cycles = 25
    dp = ds.from_host(pb, "cuda")
    g = ds.simulate(dp, p, cycles, sp.seed, sp.cfg_tag, series=True)
    torch.cuda.synchronize()
    want = oracle.simulate(pb, p, cycles, sp.seed, sp.cfg_tag, series=True)
    for k in want:
        a = g[k].cpu().numpy().astype(np.int64)
        assert np.array_equal(a, want[k].astype(np.int64)), (k, np.flatnonzero(a != want[k].astype(np.int64))[:5])
    want.pop("series")
    assert want["arrived"].sum() > 0 and (want["in_slo"] > 0).any()
    # shard [80, 160) drawn and simulated on its own (global scenario index via scen_base)
    sh = synth.generate_host(sp.replace(scen_base=80, num_scen=80))
    g2 = ds.simulate(ds.from_host(sh, "cuda"), p, cycles, sp.seed, sp.cfg_tag, scen_base=80)
    torch.cuda.synchronize()
    for k in want:
        assert np.array_equal(g2[k].cpu().numpy().astype(np.int64), want[k][80:].astype(np.int64)), k


def test_aggregate_matches_host_reference(ds):
    """a8: the device aggregate (deterministic two-level reduction) equals the host reference computed
    from the same per-DNN / per-scenario outputs (integers exact, f64 sums to 1e-12)."""
    from tests.aggref import host_agg
    sp, p = synth.config(2, num_scen=700, rows_pct=20)
    pb = synth.generate_host(sp)
    g, o = run_gpu(ds, pb, p)
    want = host_agg(g)
    got = o["agg"].cpu().numpy()
    assert np.array_equal(got[5:], want[5:])
    np.testing.assert_allclose(got[:5].view(np.float64), want[:5].view(np.float64), rtol=1e-12)


def test_aggregate_of_shards_adds_up(ds):
    """a8 across shards (the multi-GPU combine): the device aggregates of two uneven global-index shards, summed
    word by word as the NCCL all-reduce does, equal the device aggregate of the whole problem -- integer words
    (counts, histograms, position-free checksum) exactly, the f64 sums to 1e-12."""
    n = 900
    sp, p = synth.config(2, num_scen=n, rows_pct=20)
    _, whole = run_gpu(ds, synth.generate_host(sp), p)
    parts = []
    for r in range(2):
        b, e = (0, 337) if r == 0 else (337, n)
        _, o = run_gpu(ds, synth.generate_host(sp.replace(scen_base=b, num_scen=e - b)), p)
        parts.append(o["agg"].cpu().numpy())
    want = whole["agg"].cpu().numpy()
    ints = parts[0][5:].view(np.uint64) + parts[1][5:].view(np.uint64)
    assert np.array_equal(ints, want[5:].view(np.uint64))
    f = parts[0][:5].view(np.float64) + parts[1][:5].view(np.float64)
    np.testing.assert_allclose(f, want[:5].view(np.float64), rtol=1e-12)


def fast_path_problem(S_tot):
    """DNNs that drive every branch of k_prof_fast (prof.cu): certificate failure (t_np = 0, so the b >= 2
    bound has no gap), RT >= 2^24 (u32 prefix range exceeded), X(L, b_hi) within 1e-4 of 2^56 on either
    side, b_hi = 1 (no certificate), an SLO below every latency (INFEASIBLE), n = 0 rows, and ordinary
    DNNs, all under the default (linear, per_request, b_min = 1) model."""
    from tests.helpers import multi_dnn_problem
    base = dict(rows=[(10, 1, 1000), (3, 2, 500), (0, 1, 0), (200, 1, 5000)], t_p=20, t_np=5, M=50000, slo=20000,
                a=300, bmax=64)
    dnns = [base,
            dict(base, t_np=0),                                                  # certificate fails
            dict(base, rows=[(3, 65535, 7)] * 260 + [(90, 1, 0)], t_p=1, t_np=1, M=1, slo=10**9),   # RT > 2^24
            # X(L, 1) = M t_p S_tot just below 2^56 (OK) and just above (OVERFLOW), both within 1e-4 of it
            dict(base, rows=[(1, 1, 0)], t_p=(2**32 - 1) // S_tot, t_np=0, M=2**24, bmax=1, slo=10**9),
            dict(base, rows=[(1, 1, 0)], t_p=(2**32 - 1) // S_tot + 1, t_np=0, M=2**24, bmax=1, slo=10**9),
            dict(base, bmax=1),
            dict(base, slo=100, a=5000),                                          # INFEASIBLE
            dict(base, rows=[(0, 2, 10), (7, 1, 0)]),
            dict(base, rows=[(i % 40 + 1, 1 + i % 3, 100 * i) for i in range(150)], t_p=7, t_np=3)]
    return multi_dnn_problem(dnns, [3, 3, 3])


@pytest.mark.parametrize("L,S_tot", [(148, 148), (100, 80), (100, 148), (200, 200), (255, 256)])
def test_fast_path_branches_parity(ds, L, S_tot):
    pb = fast_path_problem(S_tot)
    p = Params(L=L, S_tot=S_tot, mem_mode=1)
    g, _ = run_gpu(ds, pb, p)
    want = oracle.evaluate(pb, p)
    assert_parity(g, want, where=f"fast L={L} S_tot={S_tot}")
    assert oracle.OVERFLOW in want["status"].tolist() and oracle.INFEASIBLE in want["status"].tolist()


@pytest.mark.parametrize("S_tot", [200, 256])
def test_wide_smcount_parity(ds, S_tot):
    """S_tot > 159 takes the 9-widths-per-lane fast kernel (k_prof_fast<9>)."""
    sp, p = synth.config(2, num_scen=60, rows_pct=15)
    pb = synth.generate_host(sp)
    p = p.replace(L=min(255, S_tot), S_tot=S_tot, ideal=0)
    g, _ = run_gpu(ds, pb, p)
    assert_parity(g, oracle.evaluate(pb, p), ideal=False, where=f"S_tot={S_tot}")


def run_compare(ds, pb, p):
    dp = ds.from_host(pb, "cuda")
    o = ds.eval_batch(dp, p)
    c = ds.compare(dp, p, o["demand"], o["batch"], o["alloc_q16"])
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in c.items()}, ds.to_numpy(o, pb.num_scen, pb.num_dnn)


def assert_compare_parity(g, want, where=""):
    for k in ("u", "thr", "jain"):
        a, b = g[k], want[k]
        np.testing.assert_allclose(a, b, rtol=1e-6, atol=0, err_msg=f"{where} {k}")
        assert np.array_equal(a, b), f"{where} {k}: not bit-identical"


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_compare_parity(ds, cfg):
    """O9 comparison schedulers (dstack_compare) vs the oracle, every scheduler column, bit-identical."""
    sp, p = synth.config(cfg, num_scen=None if cfg == 1 else 120, rows_pct=20)
    pb = synth.generate_host(sp)
    g, ev = run_compare(ds, pb, p)
    want = oracle.compare(pb, p)
    assert_compare_parity(g, want, where=f"config {cfg}")
    ok = ev["T_us"] > 0
    assert np.array_equal(g["u"][ok, 0], ev["u"][ok])      # the D-STACK column is the eval path's session


def test_compare_parity_edges(ds):
    for p in (Params(L=100, S_tot=148), Params(L=148, S_tot=148, mem_mode=2)):
        pb = edge_problem()
        g, _ = run_compare(ds, pb, p)
        assert_compare_parity(g, oracle.compare(pb, p), where="edge")
    pb = fast_path_problem(148)
    g, _ = run_compare(ds, pb, Params(L=148, S_tot=148, mem_mode=1))
    assert_compare_parity(g, oracle.compare(pb, Params(L=148, S_tot=148, mem_mode=1)), where="fast")


def test_compare_config3_sampled(ds):
    """Config 3 at full size in the bench configuration; 150 scenarios re-drawn on the host for the oracle."""
    sp, p = synth.config(3)
    g = synth.generate_device(sp, "cuda")
    dp = ds.from_device_dict(g)
    o = ds.eval_batch(dp, p)
    c = ds.compare(dp, p, o["demand"], o["batch"], o["alloc_q16"])
    torch.cuda.synchronize()
    idx = np.random.default_rng(11).choice(sp.num_scen, 150, replace=False)
    pb = synth.sample(sp, idx)
    want = oracle.compare(pb, p)
    got = {k: v[torch.as_tensor(idx, device=v.device)].cpu().numpy() for k, v in c.items()}
    assert_compare_parity(got, want, where="config3 sample")


# ---------------------------------------------------------------- F1 below-knee fallback ---

@pytest.mark.parametrize("variant", ["cfg4", "cfg4_reconf0", "cfg2_verbatim148", "cfg4_batching"])
def test_below_knee_parity(ds, variant):
    """F1 (DSTACK_FLAG_BELOW_KNEE) through dstack_eval_batch: every output, including the
    per-scenario below-knee counts, bit-exact against the oracle."""
    if variant.startswith("cfg4"):
        sp, p = synth.config(4, num_scen=100, variant="batching" if variant == "cfg4_batching" else "default")
    else:
        sp, p = synth.config(2, num_scen=150, rows_pct=40)
        p = p.replace(mem_mode=2, L=148)
    p = p.replace(below_knee=1, reconf_us=0 if variant == "cfg4_reconf0" else 100)
    pb = synth.generate_host(sp)
    g, _ = run_gpu(ds, pb, p)
    want = oracle.evaluate(pb, p)
    assert_parity(g, want, where=f"below-knee {variant}")
    if variant.startswith("cfg4"):
        assert want["below"].sum() > 0


def test_below_knee_split_path_and_edges(ds):
    """F1 through the call-by-call path (dstack_schedule_cycle recomputes sum R and sum R d from the rows) and on
    the hand-made edge cases."""
    sp, p = synth.config(4, num_scen=60)
    p = p.replace(below_knee=1)
    pb = synth.generate_host(sp)
    dp = ds.from_host(pb, "cuda")
    o = ds.alloc_outputs(dp, agg=False)
    ws = ds.Workspace(ds.workspace_size(dp, p), dp.device)
    ds.batch_opt(dp, p, out=o)
    ds.wmaxmin(dp.scen_dnn_off, p.L, o["demand"], out=o["alloc_q16"])
    ds.schedule_cycle(dp, p, o["demand"], o["batch"], o["alloc_q16"], out=o, ws=ws)
    torch.cuda.synchronize()
    want = oracle.evaluate(pb, p)
    assert_parity(ds.to_numpy(o, pb.num_scen, pb.num_dnn), want, where="below-knee split")
    assert want["below"].sum() > 0
    pe = edge_problem()
    for q in (Params(L=100, S_tot=148, ideal=1, below_knee=1), Params(L=148, S_tot=148, mem_mode=2, below_knee=1)):
        g, _ = run_gpu(ds, pe, q)
        assert_parity(g, oracle.evaluate(pe, q), where="below-knee edge")


# ---------------------------------------------------------------- F3 online knee discovery ---

def test_knee_probe_parity(ds):
    """F3 (dstack_knee_probe): knee found by the binary search from 30%, its step count and the
    statuses bit-exact against the oracle, in every model mode, with L < S_tot, L = S_tot and L > S_tot."""
    sp, p = synth.config(2, num_scen=80, rows_pct=30)
    pb = synth.generate_host(sp)
    dp = ds.from_host(pb, "cuda")
    pbt = synth.generate_host(sp.replace(threads=1))
    dpt = ds.from_host(pbt, "cuda")
    for pp in (p, p.replace(mem_mode=2), p.replace(mem_mode=0, L=148), p.replace(L=200, S_tot=148),
               p.replace(par_mode=1, wse_mode=1), p.replace(wse_mode=1, L=37)):
        pbx, dpx = (pbt, dpt) if pp.par_mode == 1 else (pb, dp)
        for b in (1, 3, 16, 64):
            k, pr, st = ds.knee_probe(dpx, pp, b)
            ko, pro, sto = oracle.knee_probe(pbx, pp, b)
            assert np.array_equal(st.cpu().numpy(), sto), (b, pp)
            assert np.array_equal(k.cpu().numpy().view(np.uint16), ko), (b, pp)
            assert np.array_equal(pr.cpu().numpy(), pro), (b, pp)
    pe = edge_problem()
    dpe = ds.from_host(pe, "cuda")
    q = Params(L=100, S_tot=148)
    k, pr, st = ds.knee_probe(dpe, q, 2)
    ko, pro, sto = oracle.knee_probe(pe, q, 2)
    assert np.array_equal(st.cpu().numpy(), sto) and np.array_equal(k.cpu().numpy().view(np.uint16), ko)
    assert np.array_equal(pr.cpu().numpy(), pro)


# ---------------------------------------------------------------- F4 multi-GPU cluster ---

def run_cluster(ds, pb, p, G):
    dp = ds.from_host(pb, "cuda")
    o = ds.eval_batch(dp, p)
    c = ds.cluster(dp, p, G, o["demand"], o["batch"])
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in c.items()}


@pytest.mark.parametrize("cfg,G", [(1, 4), (2, 1), (2, 3), (4, 4), (4, 8), (3, 2)])
def test_cluster_parity(ds, cfg, G):
    """F4 (dstack_cluster): every policy's U and throughput bit-identical to the oracle."""
    sp, p = synth.config(cfg, num_scen=None if cfg == 1 else 100, rows_pct=30)
    pb = synth.generate_host(sp)
    g = run_cluster(ds, pb, p, G)
    want = oracle.cluster(pb, p, G)
    for k in ("u", "thr"):
        np.testing.assert_allclose(g[k], want[k], rtol=1e-6, atol=0, err_msg=f"cluster {cfg} G={G} {k}")
        assert np.array_equal(g[k], want[k]), (cfg, G, k)


def test_cluster_edges_and_config3_sample(ds):
    pe = edge_problem()
    for p in (Params(L=100, S_tot=148), Params(L=148, S_tot=148, mem_mode=2)):
        g = run_cluster(ds, pe, p, 4)
        want = oracle.cluster(pe, p, 4)
        assert np.array_equal(g["u"], want["u"]) and np.array_equal(g["thr"], want["thr"])
    sp, p = synth.config(3)
    gd = synth.generate_device(sp, "cuda")
    dp = ds.from_device_dict(gd)
    o = ds.eval_batch(dp, p)
    c = ds.cluster(dp, p, 4, o["demand"], o["batch"])
    torch.cuda.synchronize()
    idx = np.random.default_rng(12).choice(sp.num_scen, 100, replace=False)
    want = oracle.cluster(synth.sample(sp, idx), p, 4)
    for k in ("u", "thr"):
        got = c[k][torch.as_tensor(idx, device=c[k].device)].cpu().numpy()
        assert np.array_equal(got, want[k]), k


# ---------------------------------------------------------------- compact row transport ---

def test_unpack_nr_round_trip_and_eval(ds):
    """dstack_unpack_nr expands the compact rows (n | R << 12) into exactly the wide arrays, and the path evaluated
    on the expanded rows equals the path on the original rows (config 2 sample, ragged row count)."""
    sp, p = synth.config(2, num_scen=300, rows_pct=40)
    g = synth.generate_device(sp, "cuda")
    R = int(g["dnn_row_off"][-1].item())
    nr = ds.pack_nr(g["n"][:R].cpu(), g["r"][:R].cpu())
    assert nr is not None
    nr_d = torch.zeros(R + 16, dtype=torch.int16, device="cuda")
    nr_d[:R] = nr.cuda()
    n2 = torch.full((R + 16,), -1, dtype=torch.int32, device="cuda")
    r2 = torch.full((R + 16,), -1, dtype=torch.int16, device="cuda")
    ds.unpack_nr(nr_d, n2, r2, R)
    torch.cuda.synchronize()
    assert torch.equal(n2[:R], g["n"][:R]) and torch.equal(r2[:R], g["r"][:R])
    assert int((n2[R:] != -1).sum()) == 0 and int((r2[R:] != -1).sum()) == 0   # nothing written past the rows
    o1 = ds.eval_batch(ds.from_device_dict(g), p)
    g2 = dict(g, n=n2, r=r2)
    o2 = ds.eval_batch(ds.from_device_dict(g2), p)
    torch.cuda.synchronize()
    for k in ("demand", "batch", "alloc_q16", "runs", "served", "u", "thr", "u_ideal"):
        assert torch.equal(o1[k], o2[k]), k
    assert ds.pack_nr(torch.tensor([4096], dtype=torch.int32), torch.tensor([1], dtype=torch.int16)) is None


def test_long_sessions_parity(ds):
    """Sessions of 1001..4000 slots (SLOs x4: 100-400 ms): k_cycle's long-run occupancy paths -- sessions over 1024
    slots go through the queued full-buffer pass, shorter ones in the same call through the small-buffer pass -- and
    the ideal scheduler over longer horizons, against the oracle; with and without F1."""
    sp, p = synth.config(2, num_scen=60, rows_pct=30)
    pb = synth.generate_host(sp)
    off = pb.scen_dnn_off
    for sc in range(0, pb.num_scen, 2):   # every other scenario: SLOs x4 (the rest keep sessions <= 1000 slots)
        pb.slo_us[off[sc]:off[sc + 1]] *= 4
    for q in (p, p.replace(below_knee=1), p.replace(L=148, ideal=0)):
        g, _ = run_gpu(ds, pb, q)
        want = oracle.evaluate(pb, q)
        assert_parity(g, want, ideal=bool(q.ideal), where=f"long sessions {q}")
        ns = want["T_us"] // q.slot_us
        assert (ns > 1024).any() and ((ns > 0) & (ns <= 1024)).any()   # both k_cycle passes


def test_long_sessions_compare_cluster_simulate(ds):
    """The other session users (O9 compare, F4 cluster, a7 simulate) on sessions of more than 1024 slots."""
    sp, p = synth.config(2, num_scen=40, rows_pct=30)
    pb = synth.generate_host(sp)
    pb.slo_us[:] = pb.slo_us * 4
    g, _ = run_compare(ds, pb, p)
    assert_compare_parity(g, oracle.compare(pb, p), where="long compare")
    gc = run_cluster(ds, pb, p, 3)
    wc = oracle.cluster(pb, p, 3)
    assert np.array_equal(gc["u"], wc["u"]) and np.array_equal(gc["thr"], wc["thr"])
    sp5, p5 = synth.config(5, num_scen=40, rows_pct=30)
    pb5 = synth.generate_host(sp5)
    pb5.slo_us[:] = pb5.slo_us * 4
    r = ds.simulate(ds.from_host(pb5, "cuda"), p5, 6, sp5.seed, sp5.cfg_tag)
    torch.cuda.synchronize()
    want = oracle.simulate(pb5, p5, 6, sp5.seed, sp5.cfg_tag)
    for k in want:
        assert np.array_equal(r[k].cpu().numpy().astype(np.int64), want[k].astype(np.int64)), k


def test_wide_scenarios_parity(ds):
    """Scenarios of 17..32 DNNs (every lane of the warp-per-scenario kernels holds a DNN): eval with the ideal
    scheduler, F1, O9 compare and F4 cluster against the oracle."""
    sp, p = synth.config(2, num_scen=40, rows_pct=15)
    sp = sp.replace(ndnn_min=17, ndnn_max=32)
    pb = synth.generate_host(sp)
    assert pb.num_dnn > 40 * 20
    for q in (p, p.replace(below_knee=1, ideal=0), p.replace(L=148, S_tot=148)):
        g, _ = run_gpu(ds, pb, q)
        assert_parity(g, oracle.evaluate(pb, q), ideal=bool(q.ideal), where=f"wide scenarios {q}")
    gcmp, _ = run_compare(ds, pb, p)
    assert_compare_parity(gcmp, oracle.compare(pb, p), where="wide compare")
    gc = run_cluster(ds, pb, p, 8)
    wc = oracle.cluster(pb, p, 8)
    assert np.array_equal(gc["u"], wc["u"]) and np.array_equal(gc["thr"], wc["thr"])
    sp5, p5 = synth.config(5, num_scen=30, rows_pct=15)
    sp5 = sp5.replace(ndnn_min=17, ndnn_max=32)
    pb5 = synth.generate_host(sp5)
    r = ds.simulate(ds.from_host(pb5, "cuda"), p5, 8, sp5.seed, sp5.cfg_tag)
    torch.cuda.synchronize()
    want = oracle.simulate(pb5, p5, 8, sp5.seed, sp5.cfg_tag)
    for k in want:
        assert np.array_equal(r[k].cpu().numpy().astype(np.int64), want[k].astype(np.int64)), k
    k, pr, st = ds.knee_probe(ds.from_host(pb, "cuda"), p, 2)
    ko, pro, sto = oracle.knee_probe(pb, p, 2)
    assert np.array_equal(k.cpu().numpy().view(np.uint16), ko) and np.array_equal(pr.cpu().numpy(), pro)


def test_empty_problem_calls(ds):
    """Zero scenarios / zero DNNs: every entry point returns OK without touching outputs."""
    pb = synth.make_problem([0], [0], [], [], [], [], [], [], [], [], [])
    dp = ds.from_host(pb, "cuda")
    for q in (Params(L=100, S_tot=148, ideal=1), Params(L=148, S_tot=148, below_knee=1)):
        o = ds.eval_batch(dp, q)
        torch.cuda.synchronize()
        agg = ds.agg_to_dict(o["agg"])
        assert agg["n_scen"] == 0 and agg["n_dnn"] == 0
    p = Params(L=100, S_tot=148)
    ds.knee(dp, p, 1); ds.knee_probe(dp, p, 1); ds.batch_opt(dp, p)
    ds.compare(dp, p, torch.zeros(1, dtype=torch.int16, device="cuda"), torch.zeros(1, dtype=torch.uint8, device="cuda"),
               torch.zeros(1, dtype=torch.int32, device="cuda"))
    ds.cluster(dp, p, 4, torch.zeros(1, dtype=torch.int16, device="cuda"), torch.zeros(1, dtype=torch.uint8, device="cuda"))
    ds.simulate(dp, p, 3, 1, 5)
    torch.cuda.synchronize()


def test_unpack_w5_round_trip(ds):
    """dstack_unpack_w5 (5-byte rows) expands exactly into the wide n / r / d arrays (ragged row count)."""
    sp, p = synth.config(3, num_scen=200, rows_pct=40)
    g = synth.generate_device(sp, "cuda")
    R = int(g["dnn_row_off"][-1].item())
    nn = g["n"][:R].to(torch.int64) & 0xFFFFFFFF
    rr = g["r"][:R].to(torch.int64) & 0xFFFF
    dd = g["d"][:R].to(torch.int64) & 0xFFFFFFFF
    assert int(nn.max()) < 4096 and int(rr.max()) <= 4 and int(dd.max()) < (1 << 26)
    w = torch.zeros(R + 16, dtype=torch.int64, device="cuda")
    w[:R] = dd | ((rr - 1) << 26) | ((nn >> 8) << 28)
    w = w.to(torch.int32)
    lo = torch.zeros(R + 16, dtype=torch.uint8, device="cuda")
    lo[:R] = (nn & 255).to(torch.uint8)
    n2 = torch.full((R + 16,), -1, dtype=torch.int32, device="cuda")
    r2 = torch.full((R + 16,), -1, dtype=torch.int16, device="cuda")
    d2 = torch.full((R + 16,), -1, dtype=torch.int32, device="cuda")
    ds.unpack_w5(w, lo, n2, r2, d2, R)
    torch.cuda.synchronize()
    assert torch.equal(n2[:R], g["n"][:R]) and torch.equal(r2[:R], g["r"][:R]) and torch.equal(d2[:R], g["d"][:R])
    assert int((n2[R:] != -1).sum()) == 0 and int((r2[R:] != -1).sum()) == 0 and int((d2[R:] != -1).sum()) == 0


def maxthr_workload(n, variant="default", rows_pct=20):
    """Config-2 mixes (<= 5 DNNs) with 2.5 ms slots: sessions of 10-40 slots, run lengths of a few slots -- the
    small instances the exact max-throughput search (O9b) is for."""
    sp, p = synth.config(2, num_scen=n, rows_pct=rows_pct, variant=variant)
    sp = sp.replace(slot_us=2500, slo_min_slots=10, slo_max_slots=40, ndnn_max=5)
    return sp, p.replace(slot_us=2500, ideal=0)


@pytest.mark.parametrize("variant", ["default", "batching"])
def test_max_throughput_parity(ds, variant):
    """O9b (dstack_max_throughput) against the oracle's exhaustive search: served count and status bit-exact per
    scenario; every OK scenario serves at least D-STACK's own session count."""
    sp, p = maxthr_workload(300 if variant == "default" else 120, variant)
    pb = synth.generate_host(sp)
    dp = ds.from_host(pb, "cuda")
    o = ds.eval_batch(dp, p)
    served, st = ds.max_throughput(dp, p, o["demand"], o["batch"], o["alloc_q16"])
    torch.cuda.synchronize()
    want = oracle.maxthr(pb, p)
    assert np.array_equal(st.cpu().numpy(), want["status"])
    assert np.array_equal(served.cpu().numpy().astype(np.int64), want["served"])
    ok = want["status"] == oracle.OK
    assert ok.sum() > 0.5 * pb.num_scen
    g = ds.to_numpy(o, pb.num_scen, pb.num_dnn)
    dst = np.rint(g["thr"] * g["T_us"] / 1e6).astype(np.int64)
    assert (want["served"][ok] >= dst[ok]).all()
    if variant == "batching":
        assert (want["served"][ok] > dst[ok]).any()


def test_max_throughput_caps(ds):
    """O9b beyond its exact-search caps (100 us slots: run lengths of ~60 slots, so 3+ DNNs exceed 8192 states; and
    9-12 DNN mixes exceed 8 active DNNs): the same INVALID / OK split and counts as the oracle."""
    sp, p = synth.config(2, num_scen=60, rows_pct=20)
    sp = sp.replace(ndnn_min=2, ndnn_max=12)
    p = p.replace(ideal=0)
    pb = synth.generate_host(sp)
    dp = ds.from_host(pb, "cuda")
    o = ds.eval_batch(dp, p)
    served, st = ds.max_throughput(dp, p, o["demand"], o["batch"], o["alloc_q16"])
    torch.cuda.synchronize()
    want = oracle.maxthr(pb, p)
    assert np.array_equal(st.cpu().numpy(), want["status"])
    assert np.array_equal(served.cpu().numpy().astype(np.int64), want["served"])
    assert (want["status"] == oracle.INVALID).any() and (want["status"] == oracle.OK).any()


@pytest.mark.parametrize("leg", ["compare", "cluster", "knee_probe", "below_knee", "max_throughput", "simulate"])
def test_random_profiles_legs_parity(ds, leg):
    """The §8 "next" rows (O9, F4, F3, F1, O9b) and a7 on the adversarial random profiles of
    test_random_profiles_parity: every output bit-exact against the oracle."""
    seed = {"compare": 11, "cluster": 12, "knee_probe": 13, "below_knee": 14, "max_throughput": 15,
            "simulate": 16}[leg]
    pb = random_profile_problem(seed, S=80 if leg == "max_throughput" else 200)
    p = Params(L=100, S_tot=148, ideal=0)
    dp = ds.from_host(pb, "cuda")
    if leg == "knee_probe":
        for pp in (p, p.replace(mem_mode=2), p.replace(wse_mode=1, L=148)):
            for b in (1, 7, 64):
                k, pr, st = ds.knee_probe(dp, pp, b)
                ko, pro, sto = oracle.knee_probe(pb, pp, b)
                assert np.array_equal(st.cpu().numpy(), sto), (b, pp)
                assert np.array_equal(k.cpu().numpy().view(np.uint16), ko), (b, pp)
                assert np.array_equal(pr.cpu().numpy(), pro), (b, pp)
        return
    if leg == "below_knee":
        p = p.replace(below_knee=1)
        g, _ = run_gpu(ds, pb, p)
        assert_parity(g, oracle.evaluate(pb, p, nthreads=8), ideal=False, where="random below-knee")
        return
    if leg == "simulate":
        lam = np.random.default_rng(seed).integers(0, 201, pb.num_dnn).astype(np.int32)   # 0-200 % offered load
        pb = dataclasses.replace(pb, lam_pct=lam)
        dp = ds.from_host(pb, "cuda")
        g = ds.simulate(dp, p, 12, 99, 5, series=True)
        torch.cuda.synchronize()
        want = oracle.simulate(pb, p, 12, 99, 5, series=True)
        for k in want:
            a = g[k].cpu().numpy().astype(np.int64)
            assert np.array_equal(a, want[k].astype(np.int64)), (k, np.flatnonzero(a != want[k].astype(np.int64))[:5])
        return
    o = ds.eval_batch(dp, p)
    if leg == "compare":
        c = ds.compare(dp, p, o["demand"], o["batch"], o["alloc_q16"])
        torch.cuda.synchronize()
        assert_compare_parity({k: v.cpu().numpy() for k, v in c.items()}, oracle.compare(pb, p, nthreads=8),
                              where="random compare")
    elif leg == "cluster":
        for G in (1, 3, 8):
            c = ds.cluster(dp, p, G, o["demand"], o["batch"])
            torch.cuda.synchronize()
            want = oracle.cluster(pb, p, G, nthreads=8)
            for k in ("u", "thr"):
                assert np.array_equal(c[k].cpu().numpy(), want[k]), (G, k)
    else:
        served, st = ds.max_throughput(dp, p, o["demand"], o["batch"], o["alloc_q16"])
        torch.cuda.synchronize()
        want = oracle.maxthr(pb, p, nthreads=8)
        assert np.array_equal(st.cpu().numpy(), want["status"])
        assert np.array_equal(served.cpu().numpy().astype(np.int64), want["served"])


@pytest.mark.parametrize("S_tot", [1, 2, 7, 8, 9, 16, 17, 63, 149, 255])
def test_knee_search_sm_counts_parity(ds, S_tot):
    """k_prof_lane's a2/a3 searches (PA rows with PPA checkpoints every 8 widths, binary searches over the levels and
    the certificate's segments) at SM counts around the checkpoint and word boundaries, with every width a level
    (L = S_tot), coarse levels (L < S_tot) and repeated widths (L > S_tot), on adversarial random profiles."""
    pb = random_profile_problem(40 + S_tot, S=60, S_tot=S_tot)
    for L in sorted({S_tot, max(1, S_tot // 3), min(255, 2 * S_tot)}):
        p = Params(L=L, S_tot=S_tot, ideal=0)
        g, _ = run_gpu(ds, pb, p)
        assert_parity(g, oracle.evaluate(pb, p, nthreads=8), ideal=False, where=f"L={L} S_tot={S_tot}")
