"""StreamingRunner / simulate_pulse / metrics (reference harness.py:221-334,
metrics.py) -- host logic on CPU, the device path under -m gpu."""

import math

import numpy as np
import pytest

import paper_2603_08582_b200 as sf
from paper_2603_08582_b200 import metrics
import oracle.sarfista_oracle as orc


def test_metrics_match_reference_semantics():
    rec = np.array([3.0, -3.0, 1.0, 1.0])
    mask = np.array([True, True, False, False])
    r = metrics.snr_db(rec, mask)
    assert r.snr_db == pytest.approx(20 * math.log10(3.0))
    assert metrics.snr_db(np.array([1.0, 0.0]), np.array([True, False])).snr_db == math.inf
    assert metrics.snr_db(np.zeros(2), np.array([True, False])).snr_db == 0.0
    with pytest.raises(ValueError):
        metrics.snr_db(rec, np.ones(4, bool))
    assert metrics.count_large(np.array([0.1, -0.03, 0.01]), 2e-2) == 2
    with pytest.raises(ValueError):
        metrics.count_large([1.0], 0.0)
    mo = metrics.memory_values(metrics.Method.ONLINE_FISTA, 10, 16, 4, 3).values_stored
    mb = metrics.memory_values(metrics.Method.BATCH_FISTA, 10, 16, 4, 3).values_stored
    assert mo == 10 * 17 + 20 * 11 and mb == 10 * 17 + 24 * (1 + 10 + 4)


@pytest.mark.gpu
def test_simulated_echoes_match_dense_forward_model():
    rng = np.random.default_rng(5)
    grid = sf.SceneGrid(12, reflectivity=rng.standard_normal(144))
    omega = sf.angular_frequencies(16, 1.0e10, 5.0e8)
    pos = np.array([[8660.254, 100.0, 5000.0], [8000.0, -3000.0, 5000.0]])
    d = sf.simulate_echoes(grid, pos, omega)
    for k in range(2):
        F = orc.forward_matrix(omega, pos[k], orc.pixel_positions(12))
        ref = F @ grid.reflectivity
        assert np.max(np.abs(d[k] - ref)) <= 1e-10 * np.max(np.abs(ref))


@pytest.mark.gpu
def test_streaming_runner_tracks_reference_loop():
    from paper_2603_08582_b200.workload import SMALL, generate

    wl = generate(SMALL["small"])
    grid = sf.SceneGrid(wl.grid.side_pixels, wl.grid.pixel_spacing, wl.grid.center,
                        reflectivity=np.abs(wl.rho))
    cfg = sf.SolverConfig(lam_rel=wl.cfg.lam_rel, inner_steps=wl.cfg.steps)
    run = sf.StreamingRunner(cfg, grid, wl.dictionary, truth=np.abs(wl.rho))
    rows = []
    for k in range(wl.cfg.n_pulses):
        geo = sf.PulseGeometry(k, wl.positions[k], wl.omega)
        p = sf.GeometricPulse(wl.d[k], geo, sf.NoiseCovariance(sigma2=wl.sigma2), wl.grid,
                              wl.dictionary)
        rows.append(run.process(None, p, k + 1))
    # the engine loop's own results (same pulses, same solver) are the reference here
    stats = sf.SufficientStatistics.empty(wl.m_atoms)
    state = sf.SolverState(np.zeros(wl.m_atoms), 1.0, stats)
    for k in range(wl.cfg.n_pulses):
        geo = sf.PulseGeometry(k, wl.positions[k], wl.omega)
        p = sf.GeometricPulse(wl.d[k], geo, sf.NoiseCovariance(sigma2=wl.sigma2), wl.grid,
                              wl.dictionary)
        st = sf.accumulate(state.stats, p)
        state = sf.online_fista_pulse(sf.SolverState(state.c_hat, state.momentum_t, st), cfg)
    assert np.array_equal(run.state.c_hat, state.c_hat)
    assert rows[-1].n_large == sf.count_large(state.c_hat)
    assert rows[-1].pulse_index == wl.cfg.n_pulses
    assert run.bp.pulse_count == wl.cfg.n_pulses
    assert np.isfinite(rows[-1].snr_bp_db)


@pytest.mark.gpu
def test_streaming_runner_rows_match_reference_harness():
    """Every per-pulse TraceRow, residual() and converged() of StreamingRunner
    (device metrics, sf_pulse_metrics) against the reference's own
    StreamingRunner run on the same pulses (tests/golden/harness.npz,
    harness.py:282-318): n_large exact, SNRs to 1e-4 dB (the BP SNR to 1e-9 dB),
    memory counts exact, residual to 1e-5 relative."""
    from types import SimpleNamespace

    from conftest import golden
    from paper_2603_08582_b200.dictionary import EdgeletDictionary

    g = golden("harness.npz")
    side = int(g["side"][0])
    rows = g["rows"]
    dic = EdgeletDictionary(g["ell_idx"], g["ell_w"], side * side, side)
    grid = sf.SceneGrid(side, reflectivity=g["truth"])
    cfg = SimpleNamespace(l_floor=1e-12, large_coeff_threshold=2e-2,
                          ideal_coeff_count=int(rows[-1, 1]), strict_count_termination=False,
                          residual_tol=float(rows[-1, 7]) * 1.01,
                          solver_config=lambda: sf.SolverConfig(lam=float(g["lam"][0]),
                                                                inner_steps=int(g["steps"][0])))
    run = sf.StreamingRunner(cfg, grid, dic)
    cov = sf.NoiseCovariance(sigma2=float(g["sigma2"][0]))
    for k in range(rows.shape[0]):
        geo = sf.PulseGeometry(k, g["positions"][k], g["omega"])
        r = run.process(None, sf.GeometricPulse(g["d"][k], geo, cov, grid, dic), k + 1)
        ref = rows[k]
        assert r.pulse_index == int(ref[0])
        assert r.n_large == int(ref[1]), (k, r.n_large, ref[1])
        assert r.snr_online_db == pytest.approx(ref[2], abs=1e-4)
        assert r.snr_bp_db == pytest.approx(ref[3], abs=1e-9)
        assert r.gain_db == pytest.approx(ref[4], abs=1e-4)
        assert (r.memory_online, r.memory_batch) == (int(ref[5]), int(ref[6]))
        assert run.residual() == pytest.approx(ref[7], rel=1e-5)
    assert run.converged()  # ideal count reached, residual inside the tolerance
    cfg.residual_tol = float(rows[-1, 7]) * 0.99
    assert not run.converged()
    cfg.strict_count_termination = True
    assert run.converged()
    cfg.ideal_coeff_count += 1
    assert not run.converged()
    assert run.bp.pulse_count == rows.shape[0]
