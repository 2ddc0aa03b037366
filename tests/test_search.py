"""parameter search, continuation and the
multi-resolution experiment against the LIVE reference's runs
(tests/golden/search_32.json, made by tests/golden/make_golden_search.py).

CPU tests replay the reference's recorded trials through a scripted solver:
they pin the drivers' control flow (which betas are solved, in which order,
accepted or not, the star values, ladders, log format) exactly.  GPU tests
run the real device solver and check the same decisions plus the numbers
(J extrema / residual 1e-3 relative, Dice +-0.5 pp).
"""
import math
from types import SimpleNamespace

import numpy as np
import pytest

import paper_2209_08189_b200 as P
from paper_2209_08189_b200 import autoparam as AP
from paper_2209_08189_b200 import experiment as EX
from conftest import golden_json, golden_npz

RTOL = 1e-3


@pytest.fixture(scope="module")
def G():
    return golden_json("search_32.json")


class _ScriptedSolver:
    """Stands in for gauss_newton_register: checks the requested betas against
    the reference's trial sequence and returns its recorded diagnostics."""

    def __init__(self, trials):
        self.trials = list(trials)
        self.calls = []

    def __call__(self, m0, m1, cfg, v0=None):
        t = self.trials[len(self.calls)]
        assert math.isclose(cfg.beta_v, t["beta_v"], rel_tol=1e-12), (cfg.beta_v, t)
        assert math.isclose(cfg.beta_w, t["beta_w"], rel_tol=1e-12), (cfg.beta_w, t)
        self.calls.append((cfg.beta_v, cfg.beta_w, v0))
        diag = P.SolverDiagnostics(relative_residual=t["residual"], j_min=t["j_min"], j_max=t["j_max"])
        diag.iterations = [None] * (t["gn_iterations"] + 1)
        return f"v{len(self.calls)}", diag


def test_search_control_flow_matches_reference(G, monkeypatch):
    S = G["search"]
    fake = _ScriptedSolver(S["trials"])
    monkeypatch.setattr(AP, "gauss_newton_register", fake)
    res = AP.search_parameters("m0", "m1", P.RegistrationConfig(**G["registration_config"]),
                               AP.SearchConfig(**G["search_config"]))
    assert len(fake.calls) == len(S["trials"]) == res.total_solves
    assert res.beta_v_star == S["beta_v_star"] and res.beta_w_star == S["beta_w_star"]
    assert [t.accepted for t in res.trials] == [t["accepted"] for t in S["trials"]]
    assert AP.format_trial_log(res.trials, include_seconds=False) == S["log"]
    assert res.diagnostics.termination_reason == "search-complete"
    assert res.diagnostics.relative_residual == S["residual"]
    # warm starts: every trial after the first starts from the previous trial's velocity
    assert fake.calls[0][2] is None
    assert all(fake.calls[i][2] is not None for i in range(1, len(fake.calls)))


def test_continuation_control_flow_matches_reference(G, monkeypatch):
    C, S = G["continuation"], G["search"]
    trials = [{"beta_v": r[1], "beta_w": r[2], "j_min": 1.0, "j_max": 1.0, "residual": 0.0, "gn_iterations": r[3]}
              for r in C["rungs"]]
    monkeypatch.setattr(AP, "gauss_newton_register", _ScriptedSolver(trials))
    sc = AP.SearchConfig(**G["search_config"])
    _, diag = AP.continuation_register("m0", "m1", S["beta_v_star"], S["beta_w_star"],
                                       P.RegistrationConfig(**G["registration_config"]), sc)
    assert [list(r) for r in diag.rungs] == C["rungs"]
    assert AP.continuation_ladder(S["beta_v_star"], sc.beta_v_max) == C["ladder_v"]
    assert AP.continuation_ladder(S["beta_w_star"], sc.beta_w_max) == C["ladder_w"]


@pytest.mark.parametrize("star,top,want", [(1e-3, 1.0, [1.0, 0.1, 0.01, 1e-3]),
                                            (2.5e-3, 1.0, [1.0, 0.1, 0.01, 2.5e-3]),
                                            (5.0, 1.0, [5.0]),
                                            (1e-5, 1e-5, [1e-5])])
def test_continuation_ladder(star, top, want):
    got = AP.continuation_ladder(star, top)
    assert len(got) == len(want) and all(math.isclose(a, b, rel_tol=1e-12) for a, b in zip(got, want))


def test_decades_and_configs():
    assert AP._decades_down(1.0, 1e-3) == [1.0, 0.1, 0.01, 1e-3]
    assert AP._decades_down(1e-4, 3e-6)[-1] == 3e-6
    for bad in (dict(j_min_bound=0.0), dict(j_min_bound=1.0), dict(beta_v_min=2.0), dict(beta_w_min=1.0)):
        with pytest.raises(ValueError):
            AP.SearchConfig(**bad)
    assert EX.nt_for_factor(16, 4, "proportional") == 4 and EX.nt_for_factor(32, 4, "proportional") == 8
    assert EX.nt_for_factor(16, 4, "fixed") == 16
    assert EX.default_interp_order(P.make_grid((256, 256, 256))) == "cubic"
    assert EX.default_interp_order(P.make_grid((512, 256, 256))) == "linear"


def test_search_error_when_first_trial_breaches(monkeypatch):
    trials = [{"beta_v": 1.0, "beta_w": 1e-5, "j_min": 0.1, "j_max": 2.0, "residual": 0.5, "gn_iterations": 1}]
    monkeypatch.setattr(AP, "gauss_newton_register", _ScriptedSolver(trials))
    with pytest.raises(P.SearchError):
        AP.search_beta_v("m0", "m1", P.RegistrationConfig(), AP.SearchConfig())


def test_trend_table_format(G):
    E = G["experiment"]
    pre = SimpleNamespace(d_a=E["pre"][0], d_vw=E["pre"][1], d_ivw=E["pre"][2])
    rows = [EX.ExperimentRow(**{**r, "dims": tuple(r["dims"]), "seconds": 0.0}) for r in E["rows"]]
    assert EX.format_trend_table(pre, rows, include_seconds=False) == E["table"]


# ---------------------------------------------------------------- GPU parity
@pytest.fixture(scope="module")
def inputs():
    import torch
    assert torch.cuda.is_available()
    a = golden_npz("search_32.npz")
    g = P.make_grid(a["m0"].shape)
    return g, P.ScalarField(g, a["m0"]), P.ScalarField(g, a["m1"]), P.LabelMap(g, a["labels0"]), \
        P.LabelMap(g, a["labels1"])


@pytest.mark.gpu
def test_gpu_search_parameters(G, inputs):
    g, m0, m1, _, _ = inputs
    S = G["search"]
    res = P.search_parameters(m0, m1, P.RegistrationConfig(**G["registration_config"]),
                              P.SearchConfig(**G["search_config"]))
    assert [(t.beta_v, t.beta_w, t.accepted) for t in res.trials] == \
        [(t["beta_v"], t["beta_w"], t["accepted"]) for t in S["trials"]]
    assert res.beta_v_star == S["beta_v_star"] and res.beta_w_star == S["beta_w_star"]
    for t, gt in zip(res.trials, S["trials"]):
        assert abs(t.j_min / gt["j_min"] - 1) < RTOL and abs(t.j_max / gt["j_max"] - 1) < RTOL
        assert abs(t.residual / gt["residual"] - 1) < RTOL
    assert res.velocity.data.is_cuda   # the warm-start chain stays in HBM


@pytest.mark.gpu
def test_gpu_continuation(G, inputs):
    g, m0, m1, _, _ = inputs
    C, S = G["continuation"], G["search"]
    v, diag = P.continuation_register(m0, m1, S["beta_v_star"], S["beta_w_star"],
                                      P.RegistrationConfig(**G["registration_config"]),
                                      P.SearchConfig(**G["search_config"]))
    assert [r[:3] for r in diag.rungs] == [tuple(r[:3]) for r in C["rungs"]]
    assert abs(diag.relative_residual / C["relative_residual"] - 1) < RTOL
    assert abs(diag.j_min / C["j_min"] - 1) < RTOL and abs(diag.j_max / C["j_max"] - 1) < RTOL
    assert diag.termination_reason == C["reason"]


@pytest.mark.gpu
def test_gpu_experiment(G, inputs):
    g, m0, m1, l0, l1 = inputs
    E = G["experiment"]
    plan = P.ExperimentPlan(m0, m1, l0, l1, factors=(1, 2),
                            base_config=P.RegistrationConfig(beta_v=1e-2, beta_w=1e-4, n_t=4, interp_order="cubic"),
                            betas=(1e-2, 1e-4))
    pre, rows, vels = P.run_experiment(plan)
    np.testing.assert_allclose([pre.d_a, pre.d_vw, pre.d_ivw], E["pre"], rtol=1e-12)
    for r, gr, v, vl2 in zip(rows, E["rows"], vels, E["v_l2"]):
        assert (r.factor, list(r.dims), r.n_t, r.gn_iterations) == (gr["factor"], gr["dims"], gr["n_t"],
                                                                     gr["gn_iterations"])
        for k in ("j_min", "j_max", "residual"):
            assert abs(getattr(r, k) / gr[k] - 1) < RTOL, k
        for k in ("d_a", "d_vw", "d_ivw"):
            assert abs(getattr(r, k) - gr[k]) <= 0.005, k
        assert v.grid.dims == g.dims
        assert abs(float(np.linalg.norm(v.numpy())) / vl2 - 1) < 1e-2


@pytest.mark.gpu
def test_gpu_device_generator_matches_host():
    """synth.c2_problem_device (the C4 tool's 1024^3 input path) == c2_problem."""
    from paper_2209_08189_b200.synth import c2_problem, c2_problem_device
    g = P.make_grid((32, 32, 32))
    host = c2_problem(g, "linear", 4)
    dev = c2_problem_device(g, "linear", 4)
    assert torch_equal(host[2].labels, dev[2].labels) and torch_equal(host[3].labels, dev[3].labels)
    for a, b in ((host[0].values, dev[0].values), (host[1].values, dev[1].values), (host[4].data, dev[4].data)):
        assert float((a - b).abs().max()) < 1e-6


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


@pytest.mark.gpu
def test_gpu_in_bounds():
    g = P.make_grid((16, 16, 16))
    j = np.full(g.dims, 1.0, np.float32)
    j[3, 4, 5] = 0.3
    assert not P.in_bounds(P.ScalarField(g, j), 0.5) and P.in_bounds(P.ScalarField(g, j), 0.25)
    j[3, 4, 5], j[0, 0, 0] = 1.0, 3.5
    assert not P.in_bounds(P.ScalarField(g, j), 0.3) and P.in_bounds(P.ScalarField(g, j), 0.2)
    with pytest.raises(ValueError):
        P.in_bounds(P.ScalarField(g, j), 1.0)
