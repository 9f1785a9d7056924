"""Generate the golden fixtures in tests/golden/ by running the REFERENCE package.

Run in the build container (the reference tree exists only there):

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src] [--skip-cfg0]

The reference is imported read-only from its source tree with the numba path
active (its default); nothing of it is copied into this repository -- only the
numeric outputs below are saved.  Inputs of the geometric runs come from this
repository's seeded workload generator (paper_2603_08582_b200.workload) and are
stored alongside the outputs so the fixtures are self-contained.

  known.npz          splitmix64 / start vector / frequencies / delays / phase
                     matrix / reference dictionary enumeration
  kernels.npz        fista_inner on seeded LASSO problems (test_kernels.py style)
  stream_dense.npz   accumulate + online_fista_pulse over random dense pulses
                     (scalar and full-matrix covariances, conftest.py:23-41)
  power.npz          hermitian_top_eigenvalue on seeded Hermitian PSD matrices
  geom_<name>.npz    full streaming runs on small geometric workloads
  cfg0.npz           the BASELINE cfg0 stream (64 pulses, M = 5120)
  batch.npz          batch_fista (solver.py:267-291) on the geom_small pulses
  harness.npz        the reference StreamingRunner (harness.py:254-318) on the
                     geom_small pulses: every TraceRow and residual()
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def load_reference(path):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.dont_write_bytecode = True
    sys.path.insert(0, path)
    import sarfista  # noqa: F401
    from sarfista import kernels

    print("reference imported from", os.path.dirname(sarfista.__file__),
          "numba active:", kernels.NUMBA_ACTIVE)
    return sarfista


def known(sf):
    from sarfista import rng as r
    from sarfista.geometry import round_trip_delay

    out = {}
    ks = np.array([0, 1, 2, 12345, 2**63, 2**64 - 1], dtype=np.uint64)
    out["splitmix_in"] = ks
    out["splitmix_out"] = np.array([r.splitmix64(int(k)) for k in ks], dtype=np.uint64)
    out["uniform_7"] = np.array([r.counter_uniform(7, i) for i in range(64)])
    out["start_33"] = r.counter_unit_complex_vector(33)
    out["start_5120"] = r.counter_unit_complex_vector(5120)
    out["omega_64"] = sf.angular_frequencies(64, 10.0e9, 500.0e6)
    out["delay_ref"] = np.array([round_trip_delay([4000.0, 0.0, 1000.0], [0.0, 0.0, 0.0])])
    rng = np.random.default_rng(2)
    om = 2.0 * np.pi * np.linspace(9.5e9, 9.7e9, 16)
    de = 2.6e-5 + 1e-8 * rng.random(40)
    out["phase_omega"], out["phase_delays"] = om, de
    out["phase_F"] = sf.kernels.delay_phase_matrix(om, de)
    # forward matrix on the cfg0 geometry (large phases)
    grid = sf.SceneGrid(32)
    traj = sf.TrajectoryConfig(radius=1e4 * np.cos(np.pi / 6), altitude=5e3,
                               arc_start=0.0, arc_end=np.radians(30.0), num_positions=64)
    pulse = sf.pulse_at(traj, grid.center, 17, out["omega_64"])
    out["fwd_gamma"] = pulse.position
    out["fwd_F"] = sf.build_forward_matrix(pulse, grid)[::8]
    # reference dictionary enumeration (dictionary.py:109-142)
    specs = {"s16_l4_r0_90": ((4,), (0.0, np.pi / 2), 16),
             "s16_l4_r4": ((4,), tuple(k * np.pi / 4 for k in range(4)), 16),
             "s12_l3l5_r8": ((3, 5), tuple(k * np.pi / 8 for k in range(8)), 12)}
    for name, (lengths, rots, side) in specs.items():
        d = sf.build_dictionary(sf.DictionarySpec(lengths, rots, side))
        out[f"dict_{name}_atoms"] = d.atoms.astype(np.uint8)
    return out


def kernels_fixture(sf):
    out = {}
    for seed in range(5):
        rng = np.random.default_rng(seed)
        m = 24 + 40 * seed
        B = rng.standard_normal((m, m))
        gram = np.ascontiguousarray(B @ B.T / m + 0.5 * np.eye(m))
        corr = np.ascontiguousarray(rng.standard_normal(m))
        L = float(np.linalg.eigvalsh(gram)[-1])
        c0 = rng.standard_normal(m) * (seed % 2)
        tau = 1.0 / L
        c, t = sf.kernels.fista_inner(gram, corr, c0, 1.0 + seed, tau, 0.05 * tau, 37)
        out[f"p{seed}_gram"], out[f"p{seed}_corr"], out[f"p{seed}_c0"] = gram, corr, c0
        out[f"p{seed}_args"] = np.array([1.0 + seed, tau, 0.05 * tau, 37.0])
        out[f"p{seed}_c"], out[f"p{seed}_t"] = c, np.array([t])
    return out


def stream_dense(sf):
    from sarfista.solver import (NoiseCovariance, PulseMeasurement, SolverConfig, SolverState,
                                 SufficientStatistics, accumulate, online_fista_pulse)

    out = {}
    rng = np.random.default_rng(101)
    m, n_r, count = 40, 12, 7
    stats = SufficientStatistics.empty(m)
    state = SolverState.initial(m)
    for k in range(count):
        G = rng.standard_normal((n_r, m)) + 1j * rng.standard_normal((n_r, m))
        d = rng.standard_normal(n_r) + 1j * rng.standard_normal(n_r)
        if k % 3 == 2:
            Bm = rng.standard_normal((n_r, n_r)) + 1j * rng.standard_normal((n_r, n_r))
            R = Bm @ Bm.conj().T + n_r * np.eye(n_r)
            cov = NoiseCovariance(matrix=R)
            out[f"k{k}_R"] = R
            out[f"k{k}_sigma2"] = np.array([0.0])
        else:
            s2 = float(rng.uniform(0.5, 2.0))
            cov = NoiseCovariance(sigma2=s2)
            out[f"k{k}_sigma2"] = np.array([s2])
        stats = accumulate(stats, PulseMeasurement(d, G, cov))
        lam = 0.05 * float(np.abs(stats.b).max())
        state = online_fista_pulse(SolverState(state.c_hat, state.momentum_t, stats),
                                   SolverConfig(lam=lam, inner_steps=5))
        out[f"k{k}_G"], out[f"k{k}_d"] = G, d
        out[f"k{k}_A"], out[f"k{k}_b"] = stats.A, stats.b
        out[f"k{k}_L"] = np.array([stats.L])
        out[f"k{k}_c"], out[f"k{k}_t"] = state.c_hat, np.array([state.momentum_t])
        out[f"k{k}_lam"] = np.array([lam])
    out["count"] = np.array([count])
    return out


def power(sf):
    from sarfista.solver import hermitian_top_eigenvalue

    out = {}
    rng = np.random.default_rng(7)
    for i in range(6):
        n = int(rng.integers(2, 40))
        B = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        X = B @ B.conj().T
        lam, conv = hermitian_top_eigenvalue(X)
        out[f"X{i}"], out[f"lam{i}"], out[f"conv{i}"] = X, np.array([lam]), np.array([conv])
    lam, conv = hermitian_top_eigenvalue(np.diag([1.0, 0.5]), rel_tol=0.0, max_iter=3)
    out["nc_lam"], out["nc_conv"] = np.array([lam]), np.array([conv])
    return out


def geom_run(sf, cfg, trace_every=1):
    """Reference streaming loop (harness.py:282-287) on a workload from this repo."""
    from sarfista.solver import (NoiseCovariance, PulseMeasurement, SolverConfig, SolverState,
                                 SufficientStatistics, accumulate, online_fista_pulse, reconstruct)

    sys.path.insert(0, REPO)
    from paper_2603_08582_b200.workload import generate

    wl = generate(cfg)
    H = wl.dictionary.atoms
    grid = sf.SceneGrid(cfg.side)
    m = H.shape[1]
    stats = SufficientStatistics.empty(m)
    state = SolverState.initial(m)
    out = {"omega": wl.omega, "positions": wl.positions, "d": wl.d,
           "sigma2": np.array([wl.sigma2]), "ell_idx": wl.dictionary.ell_idx,
           "ell_w": wl.dictionary.ell_w, "steps": np.array([cfg.steps]),
           "lam_rel": np.array([cfg.lam_rel])}
    Ls, lams, ts, cs, cidx = [], [], [], [], []
    t0 = time.time()
    for k in range(cfg.n_pulses):
        pulse = sf.PulseGeometry(k, wl.positions[k], wl.omega)
        F = sf.build_forward_matrix(pulse, grid)
        G = sf.compose(F, H)
        stats = accumulate(stats, PulseMeasurement(wl.d[k], G, NoiseCovariance(sigma2=wl.sigma2)))
        lam = cfg.lam_rel * float(np.abs(stats.b).max())
        state = online_fista_pulse(SolverState(state.c_hat, state.momentum_t, stats),
                                   SolverConfig(lam=lam, inner_steps=cfg.steps))
        Ls.append(stats.L)
        lams.append(lam)
        ts.append(state.momentum_t)
        if (k + 1) % trace_every == 0 or k == cfg.n_pulses - 1:
            cs.append(state.c_hat.copy())
            cidx.append(k)
    out.update(L=np.array(Ls), lam=np.array(lams), t=np.array(ts), c_trace=np.array(cs),
               c_trace_idx=np.array(cidx), c_final=state.c_hat, b_final=stats.b,
               image=reconstruct(state, H), fallbacks=np.array([stats.power_iteration_fallbacks]))
    if m <= 320:
        out["A_re_final"] = stats.A.real
    print(f"  {cfg.name}: {cfg.n_pulses} pulses, M={m}, {time.time() - t0:.1f}s")
    return out


def batch(sf):
    """Reference batch oracle on all pulses of the small geometric workload."""
    from sarfista.solver import (NoiseCovariance, PulseMeasurement, SolverConfig, _pulse_increments,
                                 batch_fista, hermitian_top_eigenvalue)

    sys.path.insert(0, REPO)
    from paper_2603_08582_b200.workload import SMALL, generate

    cfg = SMALL["small"]
    wl = generate(cfg)
    H = wl.dictionary.atoms
    grid = sf.SceneGrid(cfg.side)
    pulses = []
    for k in range(cfg.n_pulses):
        F = sf.build_forward_matrix(sf.PulseGeometry(k, wl.positions[k], wl.omega), grid)
        pulses.append(PulseMeasurement(wl.d[k], sf.compose(F, H), NoiseCovariance(sigma2=wl.sigma2)))
    A = sum(_pulse_increments(p)[0] for p in pulses)
    b = sum(_pulse_increments(p)[1] for p in pulses)
    A = 0.5 * (A + A.conj().T)
    L, conv = hermitian_top_eigenvalue(A)
    lam = 0.05 * float(np.abs(b).max())
    c = batch_fista(pulses, SolverConfig(lam=lam, inner_steps=1), 40)
    # the Frobenius fallback (solver.py:281-283): the same call with the power
    # iteration reporting non-convergence
    import sarfista.solver as sv

    real_power = sv.hermitian_top_eigenvalue
    sv.hermitian_top_eigenvalue = lambda A, *a, **k: (real_power(A, *a, **k)[0], False)
    try:
        c_frob = sv.batch_fista(pulses, SolverConfig(lam=lam, inner_steps=1), 40)
    finally:
        sv.hermitian_top_eigenvalue = real_power
    return {"L": np.array([L]), "converged": np.array([conv]), "lam": np.array([lam]),
            "iterations": np.array([40]), "c": c, "b": b, "c_frob": c_frob,
            "L_frob": np.array([float(np.linalg.norm(0.5 * (A + A.conj().T), "fro"))])}


def harness(sf):
    """The reference's own per-pulse caller on the small geometric workload:
    StreamingRunner.process (harness.py:282-304) rows, residual() every pulse."""
    from types import SimpleNamespace

    from sarfista.harness import StreamingRunner
    from sarfista.solver import NoiseCovariance, PulseMeasurement, SolverConfig

    sys.path.insert(0, REPO)
    from paper_2603_08582_b200.workload import SMALL, generate

    cfg = SMALL["small"]
    wl = generate(cfg)
    H = wl.dictionary.atoms
    truth = np.abs(wl.rho)  # the reference grid holds a real, nonnegative reflectivity
    grid = sf.SceneGrid(cfg.side, reflectivity=truth)
    lam = 4e-3
    ecfg = SimpleNamespace(l_floor=1e-12, large_coeff_threshold=2e-2, ideal_coeff_count=0,
                           strict_count_termination=False, residual_tol=0.05,
                           solver_config=lambda: SolverConfig(lam=lam, inner_steps=cfg.steps))
    from sarfista.dictionary import EdgeletDictionary

    run = StreamingRunner(ecfg, grid, EdgeletDictionary(H, [], cfg.side))
    rows = []
    for k in range(cfg.n_pulses):
        pulse = sf.PulseGeometry(k, wl.positions[k], wl.omega)
        F = sf.build_forward_matrix(pulse, grid)
        meas = PulseMeasurement(wl.d[k], sf.compose(F, H), NoiseCovariance(sigma2=wl.sigma2))
        r = run.process(F, meas, k + 1)
        rows.append([r.pulse_index, r.n_large, r.snr_online_db, r.snr_bp_db, r.gain_db,
                     r.memory_online, r.memory_batch, run.residual()])
    return {"rows": np.array(rows, dtype=np.float64), "lam": np.array([lam]),
            "truth": truth, "positions": wl.positions, "omega": wl.omega, "d": wl.d,
            "sigma2": np.array([wl.sigma2]), "ell_idx": wl.dictionary.ell_idx,
            "ell_w": wl.dictionary.ell_w, "side": np.array([cfg.side]),
            "steps": np.array([cfg.steps])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--skip-cfg0", action="store_true")
    ap.add_argument("--only", default=None, help="write just this fixture (e.g. batch)")
    args = ap.parse_args()
    sf = load_reference(args.ref)
    sys.path.insert(0, REPO)
    from paper_2603_08582_b200.workload import CONFIGS, SMALL

    if args.only == "batch":
        np.savez_compressed(os.path.join(HERE, "batch.npz"), **batch(sf))
        return
    if args.only == "harness":
        np.savez_compressed(os.path.join(HERE, "harness.npz"), **harness(sf))
        return

    np.savez_compressed(os.path.join(HERE, "known.npz"), **known(sf))
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernels_fixture(sf))
    np.savez_compressed(os.path.join(HERE, "stream_dense.npz"), **stream_dense(sf))
    np.savez_compressed(os.path.join(HERE, "power.npz"), **power(sf))
    for name in ("tiny", "small", "small8", "stride2"):
        np.savez_compressed(os.path.join(HERE, f"geom_{name}.npz"), **geom_run(sf, SMALL[name]))
    if not args.skip_cfg0:
        np.savez_compressed(os.path.join(HERE, "cfg0.npz"), **geom_run(sf, CONFIGS[0], trace_every=8))
    np.savez_compressed(os.path.join(HERE, "batch.npz"), **batch(sf))
    np.savez_compressed(os.path.join(HERE, "harness.npz"), **harness(sf))
    print("fixtures written to", HERE)


if __name__ == "__main__":
    main()
