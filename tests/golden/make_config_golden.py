"""Float64 oracle fixtures for the BASELINE.json configurations (cfg0-cfg4).

Run in the build container (CPU only; the GPU box only reads the outputs):

    python tests/golden/make_config_golden.py [--configs 0 1 2 3 4]

Inputs come from this repository's seeded workload generator
(paper_2603_08582_b200.workload) and are stored in the fixture
(d, sigma^2, positions, omega), so the GPU test feeds the engine exactly what
the oracle consumed.  Outputs come from the pixel-space float64 oracle
(oracle/sarfista_oracle.py: run_workload_pixel), which is first gated here
against the M-space oracle (itself pinned to the reference's own outputs,
tests/test_oracle.py):

  cfg0  all 64 pulses; gate: M-space oracle over all 64 pulses
  cfg1  all 128 pulses; gate: M-space oracle over the first 3 pulses
  cfg2  8 of the 1024 scenes (scene ids below), all 64 pulses each
  cfg3  all 256 pulses
  cfg4  the first 16 of 512 pulses (sigma^2 from the full 512-pulse run)

Stored per pulse: L, lambda, t, power-iteration count; per traced pulse: the
coefficient vector c as (indices, values) of its nonzeros.  Images are
recomputed in the test (oracle reconstruct) from the traced c.
"""

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import sarfista_oracle as orc  # noqa: E402

from paper_2603_08582_b200.workload import CONFIGS, generate, generate_batch  # noqa: E402

CFG2_SCENES = (0, 1, 137, 500, 511, 777, 1000, 1023)
CFG4_PREFIX = 16


def trace_pulses(n, every):
    return sorted(set(range(every - 1, n, every)) | {0, n - 1})


def pack(prefix, out, hist, trace):
    out[f"{prefix}L"] = np.array(hist["L"])
    out[f"{prefix}lam"] = np.array(hist["lam"])
    out[f"{prefix}t"] = np.array(hist["t"])
    out[f"{prefix}iters"] = np.array(hist["iters"], dtype=np.int32)
    out[f"{prefix}conv"] = np.array(hist["conv"], dtype=np.int8)
    out[f"{prefix}trace_idx"] = np.array(trace, dtype=np.int32)
    nnz = [np.nonzero(hist["c"][k])[0] for k in trace]
    out[f"{prefix}c_ptr"] = np.concatenate([[0], np.cumsum([i.size for i in nnz])]).astype(np.int64)
    out[f"{prefix}c_idx"] = (np.concatenate(nnz) if nnz else np.zeros(0)).astype(np.int32)
    out[f"{prefix}c_val"] = (np.concatenate([hist["c"][k][i] for k, i in zip(trace, nnz)])
                             if nnz else np.zeros(0))


def inputs(prefix, out, wl, n):
    out[f"{prefix}positions"] = np.ascontiguousarray(wl.positions[:n])
    out[f"{prefix}d"] = np.ascontiguousarray(wl.d[:n])
    out[f"{prefix}sigma2"] = np.array([wl.sigma2])


def run(wl, n, trace):
    xyz = orc.pixel_positions(wl.cfg.side)
    return orc.run_workload_pixel(wl.omega, wl.positions, wl.d, wl.sigma2,
                                  wl.dictionary.ell_idx, wl.dictionary.ell_w, xyz, wl.cfg.steps,
                                  wl.cfg.lam_rel, n_pulses=n, trace_at=trace)


def gate(wl, n, hist):
    """M-space oracle (OracleStats: Re(A) M x M, literal accumulate) on the first n pulses."""
    xyz = orc.pixel_positions(wl.cfg.side)
    _, _, _, hm = orc.run_workload(wl.omega, wl.positions, wl.d, wl.sigma2,
                                   wl.dictionary.ell_idx, wl.dictionary.ell_w, xyz, wl.cfg.steps,
                                   wl.cfg.lam_rel, n_pulses=n, trace=True)
    errs = {
        "L": max(abs(a - b) / b for a, b in zip(hist["L"][:n], hm["L"])),
        "lam": max(abs(a - b) / b for a, b in zip(hist["lam"][:n], hm["lam"])),
        "c": max(np.linalg.norm(hist["c"][k] - hm["c"][k]) / max(np.linalg.norm(hm["c"][k]), 1e-300)
                 for k in range(n) if k in hist["c"]),
        "t_equal": all(a == b for a, b in zip(hist["t"][:n], hm["t"])),
    }
    print(f"    gate vs M-space oracle over {n} pulses: {errs}", flush=True)
    assert errs["L"] < 1e-12 and errs["lam"] < 1e-12 and errs["c"] < 1e-12 and errs["t_equal"]
    return errs


def config_fixture(ci):
    cfg = CONFIGS[ci]
    t0 = time.time()
    out = {"config": np.array([ci]), "steps": np.array([cfg.steps]),
           "lam_rel": np.array([cfg.lam_rel])}
    if ci == 2:
        scenes = generate_batch(cfg, max(CFG2_SCENES) + 1)
        wl0 = scenes[0]
        out["omega"] = wl0.omega
        out["scenes"] = np.array(CFG2_SCENES, dtype=np.int32)
        trace = trace_pulses(cfg.n_pulses, 4)
        for s in CFG2_SCENES:
            wl = scenes[s]
            _, _, _, hist = run(wl, cfg.n_pulses, trace)
            inputs(f"s{s}_", out, wl, cfg.n_pulses)
            pack(f"s{s}_", out, hist, trace)
            print(f"  cfg2 scene {s}: L {hist['L'][-1]:.6e}", flush=True)
    else:
        wl = generate(cfg)
        n = CFG4_PREFIX if ci == 4 else cfg.n_pulses
        every = {0: 1, 1: 4, 3: 8, 4: 4}[ci]
        trace = trace_pulses(n, every)
        gate_n = {0: n, 1: 3}.get(ci, 0)
        trace_run = sorted(set(trace) | set(range(gate_n)))
        _, c, t, hist = run(wl, n, trace_run)
        if gate_n:
            errs = gate(wl, gate_n, hist)
            out["gate_pulses"] = np.array([gate_n])
            out["gate_err_c"] = np.array([errs["c"]])
            out["gate_err_L"] = np.array([errs["L"]])
        out["omega"] = wl.omega
        inputs("", out, wl, n)
        pack("", out, hist, trace)
    print(f"  {cfg.name}: {time.time() - t0:.1f}s", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[0, 1, 2, 3, 4])
    args = ap.parse_args()
    for ci in args.configs:
        path = os.path.join(HERE, f"oracle_cfg{ci}.npz")
        np.savez_compressed(path, **config_fixture(ci))
        print("wrote", path, os.path.getsize(path), "bytes", flush=True)


if __name__ == "__main__":
    main()
