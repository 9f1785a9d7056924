"""CPU: pin the float64 oracle against the reference's golden vectors and known answers.

Every fixture in tests/golden/ was produced by running the reference package
itself (tests/golden/make_golden.py); the oracle must reproduce it before it is
trusted as the checker of the GPU engine.
"""

import math

import numpy as np
import pytest

import sarfista_oracle as orc
from conftest import golden, rel_l2


def test_splitmix64_known_answers():
    # rng.py reference values (reference tests/test_rng.py:12-13)
    assert orc.splitmix64(0) == 16294208416658607535
    assert orc.splitmix64(1) == 10451216379200822465
    g = golden("known.npz")
    for k, v in zip(g["splitmix_in"], g["splitmix_out"]):
        assert orc.splitmix64(int(k)) == int(v)
    assert [orc.counter_uniform(7, i) for i in range(64)] == list(g["uniform_7"])


def test_start_vector_bit_exact():
    g = golden("known.npz")
    assert np.array_equal(orc.counter_unit_complex_vector(33), g["start_33"])
    assert np.array_equal(orc.counter_unit_complex_vector(5120), g["start_5120"])


def test_geometry_known_answers():
    g = golden("known.npz")
    assert np.array_equal(orc.angular_frequencies(64, 10.0e9, 500.0e6), g["omega_64"])
    tau = orc.delays(np.array([4000.0, 0.0, 1000.0]), np.zeros((1, 3)))[0]
    assert math.isclose(tau, 2.7506399948311313e-05, rel_tol=1e-12)
    assert tau == g["delay_ref"][0]


def test_phase_matrix_matches_reference():
    g = golden("known.npz")
    F = orc.delay_phase_matrix(g["phase_omega"], g["phase_delays"])
    assert np.allclose(F, g["phase_F"], rtol=1e-12, atol=1e-12)
    # cfg0 geometry: arguments of ~4e6 rad
    xyz = orc.pixel_positions(32)
    F0 = orc.forward_matrix(g["omega_64"], g["fwd_gamma"], xyz)[::8]
    assert np.max(np.abs(F0 - g["fwd_F"])) < 1e-9


def test_fista_inner_matches_reference():
    g = golden("kernels.npz")
    for s in range(5):
        t0, tau, thresh, steps = g[f"p{s}_args"]
        c, t = orc.fista_inner(g[f"p{s}_gram"], g[f"p{s}_corr"], g[f"p{s}_c0"], t0, tau, thresh,
                               int(steps))
        assert np.allclose(c, g[f"p{s}_c"], rtol=1e-12, atol=1e-13)
        assert t == pytest.approx(g[f"p{s}_t"][0], rel=1e-15)


def test_power_iteration_matches_reference():
    g = golden("power.npz")
    for i in range(6):
        lam, conv = orc.hermitian_top_eigenvalue(g[f"X{i}"])
        assert conv == bool(g[f"conv{i}"][0])
        assert lam == pytest.approx(g[f"lam{i}"][0], rel=1e-12)
    lam, conv = orc.hermitian_top_eigenvalue(np.diag([1.0, 0.5]), rel_tol=0.0, max_iter=3)
    assert not conv and lam == pytest.approx(g["nc_lam"][0], rel=1e-15)


def test_nr_space_power_iteration_equals_m_space():
    # identical iterate sequence in the N_r-dimensional image
    rng = np.random.default_rng(3)
    for n_r, m in ((4, 30), (12, 200), (32, 257)):
        G = rng.standard_normal((n_r, m)) + 1j * rng.standard_normal((n_r, m))
        X = G.conj().T @ G
        lam_m, conv_m = orc.hermitian_top_eigenvalue(0.5 * (X + X.conj().T))
        lam_r, conv_r, _, _ = orc.top_eigenvalue_nr(G, orc.counter_unit_complex_vector(m))
        assert conv_m == conv_r
        assert lam_r == pytest.approx(lam_m, rel=1e-10)


def test_dense_stream_matches_reference():
    g = golden("stream_dense.npz")
    m = g["k0_G"].shape[1]
    st = orc.OracleStats(m, keep_complex=True)
    c, t = np.zeros(m), 1.0
    for k in range(int(g["count"][0])):
        R = g[f"k{k}_R"] if f"k{k}_R" in g else None
        s2 = None if R is not None else float(g[f"k{k}_sigma2"][0])
        orc.accumulate(st, g[f"k{k}_G"], g[f"k{k}_d"], sigma2=s2, R=R)
        assert np.allclose(st.A, g[f"k{k}_A"], rtol=1e-12, atol=1e-12)
        assert np.allclose(st.A_re, g[f"k{k}_A"].real, rtol=1e-12, atol=1e-12)
        assert np.allclose(st.b, g[f"k{k}_b"], rtol=1e-12, atol=1e-12)
        assert st.L == pytest.approx(g[f"k{k}_L"][0], rel=1e-10)
        lam = 0.05 * float(np.abs(st.b).max())
        assert lam == pytest.approx(g[f"k{k}_lam"][0], rel=1e-12)
        c, t = orc.online_fista_pulse(st, c, t, lam, 5)
        assert rel_l2(c, g[f"k{k}_c"]) < 1e-9
        assert t == g[f"k{k}_t"][0]


@pytest.mark.parametrize("name", ["tiny", "small", "small8", "stride2"])
def test_geometric_stream_matches_reference(name):
    g = golden(f"geom_{name}.npz")
    side = int(round(math.sqrt(int(g["ell_idx"].max()) + 1)))
    xyz = orc.pixel_positions(side)
    st, c, t, hist = orc.run_workload(g["omega"], g["positions"], g["d"], float(g["sigma2"][0]),
                                      g["ell_idx"], g["ell_w"], xyz, int(g["steps"][0]),
                                      float(g["lam_rel"][0]), trace=True)
    assert np.allclose(hist["L"], g["L"], rtol=1e-9)
    assert np.allclose(hist["lam"], g["lam"], rtol=1e-9)
    assert np.allclose(hist["t"], g["t"], rtol=1e-15)
    for i, k in enumerate(g["c_trace_idx"]):
        assert rel_l2(hist["c"][k], g["c_trace"][i]) < 1e-8
    assert rel_l2(c, g["c_final"]) < 1e-9
    img = orc.reconstruct(g["ell_idx"], g["ell_w"], xyz.shape[0], c)
    assert rel_l2(img, g["image"]) < 1e-9
    assert rel_l2(st.b, g["b_final"]) < 1e-12
    if "A_re_final" in g:
        assert rel_l2(st.A_re, g["A_re_final"]) < 1e-12


def test_cfg0_prefix_matches_reference():
    g = golden("cfg0.npz")
    xyz = orc.pixel_positions(32)
    n = 16
    st, c, t, hist = orc.run_workload(g["omega"], g["positions"], g["d"], float(g["sigma2"][0]),
                                      g["ell_idx"], g["ell_w"], xyz, int(g["steps"][0]),
                                      float(g["lam_rel"][0]), n_pulses=n)
    assert np.allclose(hist["L"], g["L"][:n], rtol=1e-9)
    k = list(g["c_trace_idx"]).index(n - 1)
    assert rel_l2(c, g["c_trace"][k]) < 1e-8


def test_symmetric_store_matches_direct_products():
    """SymStore (upper-triangle row panels, dgemm / dgemv) against explicit
    dot products, across panel boundaries."""
    rng = np.random.default_rng(7)
    for n, k, panel in ((1, 3, 256), (37, 5, 8), (700, 24, 256), (1500, 64, 256)):
        S = orc.SymStore(n, panel)
        ref = np.zeros((n, n))
        for _ in range(2):
            P = rng.standard_normal((k, n))
            S.rank_update(np.ascontiguousarray(P.T))
            ref += P.T @ P
        D = S.dense()
        assert np.array_equal(D, D.T)
        assert np.allclose(D, ref, rtol=1e-13, atol=1e-11)
        z = rng.standard_normal(n)
        assert np.allclose(S.matvec(z), ref @ z, rtol=1e-12, atol=1e-10)


@pytest.mark.parametrize("name", ["small", "small8", "stride2"])
def test_pixel_space_oracle_equals_m_space(name):
    """The pixel-space restatement (A = H^T B H, b = H^T beta) reproduces the
    M-space oracle and the reference's own outputs on the same pulses."""
    g = golden(f"geom_{name}.npz")
    side = int(round(math.sqrt(int(g["ell_idx"].max()) + 1)))
    xyz = orc.pixel_positions(side)
    args = (g["omega"], g["positions"], g["d"], float(g["sigma2"][0]), g["ell_idx"], g["ell_w"],
            xyz, int(g["steps"][0]), float(g["lam_rel"][0]))
    n = g["positions"].shape[0]
    stp, cp, tp, hp = orc.run_workload_pixel(*args, trace_at=range(n))
    stm, cm, tm, hm = orc.run_workload(*args, trace=True)
    assert np.allclose(hp["L"], hm["L"], rtol=1e-12)
    assert np.allclose(hp["lam"], hm["lam"], rtol=1e-12)
    assert hp["t"] == hm["t"] and hp["iters"] == hm["iters"]
    for k in range(n):
        assert rel_l2(hp["c"][k], hm["c"][k]) < 1e-11
    assert rel_l2(stp.b, stm.b) < 1e-13
    assert rel_l2(cp, g["c_final"]) < 1e-9
    assert np.allclose(hp["L"], g["L"], rtol=1e-9)


def test_pixel_space_oracle_cfg0_prefix_matches_reference():
    g = golden("cfg0.npz")
    xyz = orc.pixel_positions(32)
    n = 16
    _, c, _, hist = orc.run_workload_pixel(g["omega"], g["positions"], g["d"],
                                           float(g["sigma2"][0]), g["ell_idx"], g["ell_w"], xyz,
                                           int(g["steps"][0]), float(g["lam_rel"][0]), n_pulses=n)
    assert np.allclose(hist["L"], g["L"][:n], rtol=1e-9)
    k = list(g["c_trace_idx"]).index(n - 1)
    assert rel_l2(c, g["c_trace"][k]) < 1e-8


def test_config_fixtures_are_gated():
    """tests/golden/oracle_cfg*.npz: the pixel-space oracle was gated against the
    M-space oracle when the fixture was made (make_config_golden.py)."""
    for ci in (0, 1):
        g = golden(f"oracle_cfg{ci}.npz")
        assert int(g["gate_pulses"][0]) >= 3
        assert float(g["gate_err_c"][0]) < 1e-12 and float(g["gate_err_L"][0]) < 1e-12
