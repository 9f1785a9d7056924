"""Batched scenes (BASELINE cfg2 layout): one engine, B independent scenes per
launch.  Every scene must match a single-scene engine fed the same pulses, bit
for bit (same kernels, scene offsets only)."""

import numpy as np
import pytest

from paper_2603_08582_b200.engine import Engine
from paper_2603_08582_b200.geometry import pixel_positions
from paper_2603_08582_b200.workload import SMALL, generate_batch

pytestmark = pytest.mark.gpu


def _single(wl, pulses, precision="f16x3"):
    import torch

    eng = Engine(wl.m_atoms, len(wl.omega), wl.dictionary.ell_idx, wl.dictionary.ell_w,
                 pixel_positions(wl.grid), precision=precision)
    c = torch.zeros(wl.m_atoms, dtype=torch.float64, device="cuda")
    c2 = torch.empty_like(c)
    t = 1.0
    for k in range(pulses):
        eng.accumulate_geom(wl.positions[k], wl.omega, wl.d[k], wl.sigma2)
        t = eng.fista(c, c2, wl.cfg.steps, t, lam_rel=wl.cfg.lam_rel)
        c, c2 = c2, c
    return c.cpu().numpy(), eng.scalars()[0]


@pytest.mark.parametrize("precision", ["f16x3", "dirichlet"])
@pytest.mark.parametrize("name,B,device_inputs", [("small", 3, False), ("small", 3, True),
                                                  ("small8", 5, False), ("small8", 5, True)])
def test_batched_scenes_match_single_scene_engines(name, B, device_inputs, precision):
    import torch

    scenes = generate_batch(SMALL[name], B)
    wl0 = scenes[0]
    pulses = min(s.cfg.n_pulses for s in scenes)
    eng = Engine(wl0.m_atoms, len(wl0.omega), wl0.dictionary.ell_idx, wl0.dictionary.ell_w,
                 pixel_positions(wl0.grid), batch=B, precision=precision)
    c = torch.zeros((B, wl0.m_atoms), dtype=torch.float64, device="cuda")
    c2 = torch.empty_like(c)
    t = 1.0
    for k in range(pulses):
        g = np.stack([s.positions[k] for s in scenes])
        d = np.stack([s.d[k] for s in scenes])
        s2 = np.array([s.sigma2 for s in scenes])
        if device_inputs:
            g, d, s2 = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (g, d, s2))
            w = torch.from_numpy(wl0.omega).cuda()
        else:
            w = wl0.omega
        eng.accumulate_geom_batch(g, w, d, s2)
        t = eng.fista(c, c2, wl0.cfg.steps, t, lam_rel=wl0.cfg.lam_rel)
        c, c2 = c2, c
    cb = c.cpu().numpy()
    L, n, fb = eng.batch_scalars()
    assert (n == pulses).all() and (fb == 0).all()
    for b, wl in enumerate(scenes):
        cs, Ls = _single(wl, pulses, precision)
        assert L[b] == Ls
        assert np.array_equal(cb[b], cs)
    assert np.count_nonzero(cb) > 0


def test_batched_engine_rejects_single_scene_calls():
    scenes = generate_batch(SMALL["tiny"], 2)
    wl = scenes[0]
    eng = Engine(wl.m_atoms, len(wl.omega), wl.dictionary.ell_idx, wl.dictionary.ell_w,
                 pixel_positions(wl.grid), batch=2)
    with pytest.raises(ValueError):
        eng.accumulate_geom(wl.positions[0], wl.omega, wl.d[0], wl.sigma2)
    with pytest.raises(ValueError):
        eng.accumulate_geom_batch(np.zeros((3, 3)), wl.omega, np.zeros((2, len(wl.omega))),
                                  np.ones(2))


def test_device_batch_fista_matches_reference_batch_oracle():
    """solver.batch_fista on the device vs the reference's batch_fista (golden):
    the batch step size (matrix-free power iteration on sum_k G_k^H G_k / s^2)
    and the 40-iteration FISTA solution from zero."""
    import paper_2603_08582_b200 as sf
    from conftest import golden, rel_l2
    from paper_2603_08582_b200.workload import generate

    g = golden("batch.npz")
    wl = generate(SMALL["small"])
    pulses = [sf.GeometricPulse(wl.d[k], sf.PulseGeometry(k, wl.positions[k], wl.omega),
                                sf.NoiseCovariance(sigma2=wl.sigma2), wl.grid, wl.dictionary)
              for k in range(wl.cfg.n_pulses)]
    # the step size alone
    eng = Engine(wl.m_atoms, len(wl.omega), wl.dictionary.ell_idx, wl.dictionary.ell_w,
                 pixel_positions(wl.grid))
    lam_max, conv = eng.batch_lipschitz(wl.positions, wl.omega, [wl.sigma2] * len(pulses))
    assert conv and lam_max == pytest.approx(float(g["L"][0]), rel=1e-10)
    c = sf.batch_fista(pulses, sf.SolverConfig(lam=float(g["lam"][0]), inner_steps=1),
                       int(g["iterations"][0]))
    assert rel_l2(c, g["c"]) < 1e-6
    with pytest.raises(ValueError):
        sf.batch_fista([], sf.SolverConfig(lam=1.0), 3)
    with pytest.raises(ValueError):
        sf.batch_fista(pulses, sf.SolverConfig(lam=1.0), 0)


def test_device_batch_fista_frobenius_fallback(monkeypatch):
    """The batch oracle's Frobenius fallback (solver.py:281-283): with the power
    iteration reporting non-convergence the step size is |A|_F of the full batch
    matrix; c must match the reference's batch_fista run the same way (golden
    c_frob, tests/golden/make_golden.py)."""
    import paper_2603_08582_b200 as sf
    from conftest import golden, rel_l2
    from paper_2603_08582_b200.workload import generate

    g = golden("batch.npz")
    wl = generate(SMALL["small"])
    pulses = [sf.GeometricPulse(wl.d[k], sf.PulseGeometry(k, wl.positions[k], wl.omega),
                                sf.NoiseCovariance(sigma2=wl.sigma2), wl.grid, wl.dictionary)
              for k in range(wl.cfg.n_pulses)]
    real = Engine.batch_lipschitz
    monkeypatch.setattr(Engine, "batch_lipschitz",
                        lambda self, *a, **k: (real(self, *a, **k)[0], False))
    import paper_2603_08582_b200.solver as sv
    real_power = sv.hermitian_top_eigenvalue
    monkeypatch.setattr(sv, "hermitian_top_eigenvalue",
                        lambda A, *a, **k: (real_power(A, *a, **k)[0], False))
    c = sf.batch_fista(pulses, sf.SolverConfig(lam=float(g["lam"][0]), inner_steps=1),
                       int(g["iterations"][0]))
    assert rel_l2(c, g["c_frob"]) < 1e-6
