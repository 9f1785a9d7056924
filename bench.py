#!/usr/bin/env python
"""Online-FISTA per-pulse throughput on B200 (the BASELINE.json metric).

One step = one pulse of the hot path: device synthesis of the forward operator,
the sufficient-statistics update (closed-form pixel-space Gram, tcgen05 K~
build, N_r-space power iteration) and the warm-started FISTA inner loop.

Workload (``--config``, default 3): BASELINE configs[3] ("cfg3": 128x128 scene,
M = 81920 atoms, N_r = 256, 10 FISTA steps/pulse) -- the largest BASELINE
configuration that runs on one GPU and the one the metric's 1/2/4/8-GPU sweep
is quoted on -- as seeded synthetic inputs (paper_2603_08582_b200.workload,
SURVEY App. A).  Under torchrun (N > 1) the same single scene is sharded over
the ranks (strong scaling; one NCCL all-reduce of y_pix per FISTA step);
``--replicas`` runs one independent scene per rank instead.  ``--config 2``
runs BASELINE cfg2 (1024 scenes in one batched engine per rank).

Reported (rank 0, one JSON line)
  value     pulses/s with every pulse input already resident in HBM (device-timed,
            CUDA events on the engine stream, max over ranks; L2 flushed between
            pulses)
  e2e       pulses/s through the public API (GeometricPulse -> accumulate ->
            online_fista_pulse -> c_hat) with pinned host inputs copied in and
            the coefficient vector read back every pulse
  roofline  FISTA matvec kernel (dominant): algorithmic bytes per launch / mean
            launch time, vs MEASURED_PEAKS.json hbm_gbs
  tensor_core  the tcgen05 kernel on the default path (K~ build) against the
            bf16 peak; the closed-form Gram has no contraction
  cfg1      (N = 1, default config) the same measurements at BASELINE configs[1]
  cpu_baseline  the float64 oracle port (oracle/) on this host's cores, a
            bounded sample of the same workload

--impl reference times the reference's CPU path on this host (rank 0): the
oracle port on the same config, plus the reference package itself
(baseline/_ref, pure Python) at cfg0 as BASELINE.md's CPU-baseline plan asks.
"""

import argparse
import collections
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "online pulses/sec (update+FISTA)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--cpu-pulses", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg1 extra keys")
    ap.add_argument("--flush-l2-mb", type=int, default=128,
                    help="MiB written between timed pulses (L2 flush, > the 126 MB L2; its time "
                         "counts in the timed region; 0 = no flush). A second, unflushed timed "
                         "run is reported as l2_warm")
    ap.add_argument("--scenes", type=int, default=1024,
                    help="config 2: independent scenes per engine (BASELINE cfg2: 1024)")
    ap.add_argument("--e2e-lag", type=int, default=6,
                    help="e2e loop reads pulse k's c_hat after pulse k+lag is queued")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N>1: peer-memory exchange (CUDA IPC over NVLink, push fused into the "
                         "slot reduction; falls back to NCCL if any rank cannot set it up) or "
                         "the NCCL all-reduces")
    ap.add_argument("--share-gpu", action="store_true",
                    help="testing only: every rank on cuda:0 with the gloo backend (exercises the "
                         "N>1 code path -- sharding, peer-memory exchange, reductions -- on a "
                         "one-GPU box; the numbers mean nothing)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: one independent scene per rank instead of one sharded scene")
    return ap.parse_args()


def engine_env_guard():
    """The engine reads a few SF_* switches (debug sync, graph replay off, the
    fp64 K~ path, single-buffered state -- tests and debugging only).  A bench
    number must come from the default path: refuse to run with any set."""
    bad = sorted(k for k in os.environ if k.startswith("SF_"))
    if bad:
        sys.stderr.write(f"bench.py: refusing to run with engine switches set: {bad}\n")
        sys.exit(2)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(cfg):
    return (f"{cfg.name}: {cfg.side}x{cfg.side} scene, M={cfg.m_atoms} atoms "
            f"(identity + {cfg.n_rot} rot x len {cfg.length} edgelets"
            + (f", stride {cfg.stride}" if cfg.stride > 1 else "")
            + f"), N_r={cfg.n_freq}, {cfg.n_pulses} pulses over {cfg.arc_deg:g} deg "
            f"(timed pulses cycle through the arc), {cfg.steps} FISTA steps/pulse, "
            f"SNR {cfg.snr_db:g} dB, lambda={cfg.lam_rel}*max|b|")


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", 0.0)), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clock / throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        loaded = [r for r in rows if (num(r[6]) or 0) > 0] or rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": num(rows[0][1]), "reasons": reasons, "samples": len(loaded)}


def host_cores():
    try:
        import threadpoolctl

        info = threadpoolctl.threadpool_info()
        n = max((i.get("num_threads", 0) for i in info if i.get("user_api") == "blas"), default=0)
        if n:
            return int(n)
    except Exception:
        pass
    return os.cpu_count() or 1


# ---- CPU baselines (rank 0 only; never inside a timed GPU region) -------------------

def host_mem_available():
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def oracle_fits(m_atoms):
    """The M-space port holds Re(A) as an M x M float64 array (plus G, P)."""
    need = 8.0 * m_atoms * m_atoms * 1.15
    avail = host_mem_available()
    return avail is None or need < 0.8 * avail, need


def cpu_oracle_pulses_per_s(wl, n_pulses, warm=1):
    """Float64 oracle port (oracle/sarfista_oracle.py, the reference's M-space
    algorithm: Re(A) M x M, rank-2N_r update, N_r-space power iteration, dense
    matvec FISTA) on the host cores."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import sarfista_oracle as orc

    cfg = wl.cfg
    xyz = orc.pixel_positions(cfg.side)
    st = orc.OracleStats(wl.m_atoms)
    c, t = np.zeros(wl.m_atoms), 1.0
    total = 0.0
    done = 0
    for k in range(warm + n_pulses):
        t0 = time.perf_counter()
        F = orc.forward_matrix(wl.omega, wl.positions[k], xyz)
        G = orc.compose_ell(F, wl.dictionary.ell_idx, wl.dictionary.ell_w)
        orc.accumulate(st, G, wl.d[k], wl.sigma2)
        lam = cfg.lam_rel * float(np.abs(st.b).max())
        c, t = orc.online_fista_pulse(st, c, t, lam, cfg.steps)
        dt = time.perf_counter() - t0
        if k >= warm:
            total += dt
            done += 1
    return done / total, done, total


def reference_package_cfg0(n_pulses=4):
    """The reference package itself (baseline/_ref, pure Python + numba) on
    BASELINE cfg0: build_forward_matrix + compose + accumulate +
    online_fista_pulse per pulse (BASELINE.md CPU-baseline plan), the first
    (JIT) pulse excluded."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "sarfista")):
        return {"unavailable": "baseline/_ref not installed (see DESIGN.md section 5)"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    sys.path.insert(0, ref)
    import sarfista as rsf
    from sarfista import kernels as rk

    from paper_2603_08582_b200.workload import CONFIGS, generate

    wl = generate(CONFIGS[0])
    cfg = wl.cfg
    grid = rsf.SceneGrid(cfg.side)
    H = wl.dictionary.atoms  # the extended BASELINE dictionary as a dense N x M matrix
    stats = rsf.SufficientStatistics.empty(wl.m_atoms)
    state = rsf.SolverState(np.zeros(wl.m_atoms), 1.0, stats)
    cov = rsf.NoiseCovariance(sigma2=wl.sigma2)
    total, done = 0.0, 0
    for k in range(1 + n_pulses):
        t0 = time.perf_counter()
        pulse = rsf.PulseGeometry(k, wl.positions[k], wl.omega)
        F = rsf.build_forward_matrix(pulse, grid)
        G = rsf.compose(F, H)
        stats = rsf.accumulate(state.stats, rsf.PulseMeasurement(wl.d[k], G, cov))
        lam = cfg.lam_rel * float(np.abs(stats.b).max())
        state = rsf.online_fista_pulse(rsf.SolverState(state.c_hat, state.momentum_t, stats),
                                       rsf.SolverConfig(lam=lam, inner_steps=cfg.steps))
        dt = time.perf_counter() - t0
        if k >= 1:
            total += dt
            done += 1
    port, pdone, _ = cpu_oracle_pulses_per_s(wl, 8, warm=1)
    return {"value": done / total, "unit": "pulses/s", "cores": host_cores(),
            "numba_active": bool(rk.NUMBA_ACTIVE),
            "sample": f"pulses 1..{done} of cfg0 (pulse 0 untimed: numba JIT) through the "
                      "reference package's own build_forward_matrix / compose / accumulate / "
                      "online_fista_pulse, extended dictionary passed as a dense H",
            "port_same_host": {"value": port, "pulses": pdone,
                               "note": "the float64 oracle port on the same cfg0 pulses"}}


def run_reference(args, rank, world):
    from paper_2603_08582_b200.workload import CONFIGS, generate

    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    wl = generate(cfg)  # host forward model: the reference arm touches nothing of the engine
    n = max(1, min(args.steps, args.cpu_pulses))
    ok, need = oracle_fits(wl.m_atoms)
    if not ok:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"the float64 port needs {need / 1e9:.0f} GB of host RAM for "
                          f"{cfg.name}; MemAvailable {host_mem_available() / 1e9:.0f} GB"}), flush=True)
        return
    value, done, total = cpu_oracle_pulses_per_s(wl, n, warm=1)
    cores = host_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pulses/s",
        "n_gpus": args.gpus, "steps": done, "warmup": 1, "ms_per_step": 1e3 * total / done,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY App. A)",
        "config": {"workload": workload_desc(cfg)},
        "cpu_baseline": {"value": value, "unit": "pulses/s", "cores": cores, "kind": "port",
                         "sample": f"pulses 1..{done} of {cfg.name} after 1 untimed pulse "
                                   "through the float64 oracle port (the reference's M-space "
                                   "algorithm; the reference package itself needs ~6 live "
                                   "M x M complex128 arrays, 320 GB at this config)"},
        "e2e": {"value": value, "unit": "pulses/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_package_cfg0": reference_package_cfg0(),
    }
    print(json.dumps(line), flush=True)


# ---- the engine ---------------------------------------------------------------------

def pulse_loop(eng, g_dev, w_dev, d_dev, sigma2, idx, steps_fista, lam_rel, c, c2, t, flush=None):
    for k, j in idx:
        eng.accumulate_geom(g_dev[j], w_dev, d_dev[j], sigma2)
        t = eng.fista(c, c2, steps_fista, t, lam_rel=lam_rel)
        c, c2 = c2, c
        if flush is not None:  # evict L2 between pulses (counted in the timed region)
            flush.fill_(float(k))
    return c, c2, t


def timed(torch, stream, world, fn):
    """Device time of fn() on `stream` (CUDA events), max over ranks."""
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        ms = max_over_ranks(torch, ms, stream.device)
    return ms, out


def max_over_ranks(torch, value, dev):
    """MAX of a scalar over the ranks (device tensor for NCCL, host tensor for gloo)."""
    where = dev if torch.distributed.get_backend() == "nccl" else "cpu"
    tt = torch.tensor([value], dtype=torch.float64, device=where)
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    return float(tt.item())


def q_nnz(dictionary):
    from scipy import sparse

    idx, w = dictionary.ell_idx, dictionary.ell_w
    j, l = np.nonzero(idx >= 0)
    H = sparse.csr_matrix((w[j, l], (idx[j, l], j)), shape=(dictionary.n_pixels, idx.shape[0]))
    return int((H @ H.T).nnz)


def measure_config(args, cfg, rank, world, local, sharded, main=True):
    """One configuration through the engine: device-resident timed run (flushed
    and warm), per-kernel profile, e2e through the public API."""
    import torch

    from paper_2603_08582_b200 import _lib
    from paper_2603_08582_b200 import solver as api
    from paper_2603_08582_b200.engine import Engine
    from paper_2603_08582_b200.geometry import PulseGeometry, pixel_positions
    from paper_2603_08582_b200.workload import generate

    dev = torch.device("cuda", local)
    wl = generate(cfg, device_sim=True)  # echoes from the device simulator (host noise draws)
    M, n_r = wl.m_atoms, cfg.n_freq
    xyz = pixel_positions(wl.grid)
    n_total = args.warmup + args.steps
    idx = [(k, k % cfg.n_pulses) for k in range(n_total)]

    eng = Engine(M, n_r, wl.dictionary.ell_idx, wl.dictionary.ell_w, xyz, device=local)
    stream = torch.cuda.current_stream(dev)
    eng.set_stream(stream)
    keep = []  # peer-memory groups live as long as their engines
    exch = "none"
    if sharded:
        from paper_2603_08582_b200 import sharding

        exch, pg = sharding.shard_auto(eng, prefer=args.exchange)
        keep.append(pg)
    g_dev = torch.from_numpy(np.ascontiguousarray(wl.positions)).to(dev)
    w_dev = torch.from_numpy(np.ascontiguousarray(wl.omega)).to(dev)
    d_dev = torch.from_numpy(np.ascontiguousarray(wl.d)).to(dev)
    c = torch.zeros(M, dtype=torch.float64, device=dev)
    c2 = torch.empty_like(c)
    flush = (torch.empty(args.flush_l2_mb << 17, dtype=torch.float64, device=dev)
             if args.flush_l2_mb > 0 else None)
    loop = lambda ids, t, fl: pulse_loop(eng, g_dev, w_dev, d_dev, wl.sigma2, ids, cfg.steps,
                                         cfg.lam_rel, c, c2, t, fl)
    c, c2, t = loop(idx[:args.warmup], 1.0, flush)
    l0 = _lib.launch_count()
    ms, (c, c2, t) = timed(torch, stream, world, lambda: loop(idx[args.warmup:], t, flush))
    launches = _lib.launch_count() - l0
    units = 1 if sharded else world
    out = {"value": units * args.steps / (ms / 1e3), "ms_per_step": ms / args.steps,
           "gpu_launches": launches}
    store_bytes = eng.n_tiles_local() * 65536
    if flush is not None and store_bytes < 100e6:
        # (the warm pass continues the same state, so it is only meaningful
        # where the store can stay in L2 -- cfg0-cfg2; cfg3/cfg4 stream HBM)
        wms, (c, c2, t) = timed(torch, stream, world, lambda: loop(idx[args.warmup:], t, None))
        out["l2_warm"] = {"value": units * args.steps / (wms / 1e3), "ms_per_step": wms / args.steps,
                          "note": "the same pulses without the L2 flush between them"}
    kinds = (("gemv", _lib.K_GEMV), ("gram", _lib.K_GRAM), ("fista_loop", _lib.K_STEP),
             ("operator", _lib.K_OPERATOR), ("fista_call", _lib.K_FISTA), ("ktilde", _lib.K_KTILDE))

    def profiled(e, ids, cc, cc2, tt):
        """Per-kernel CUDA-event timing (a separate pass: events perturb the timed
        loop) and the matvec's requested tile bytes over the pulses `ids`."""
        e.profile(True)
        cc, cc2, tt = pulse_loop(e, g_dev, w_dev, d_dev, wl.sigma2, ids, cfg.steps, cfg.lam_rel,
                                 cc, cc2, tt, flush)
        torch.cuda.synchronize(dev)
        res = {name: e.profile_read(kind) for name, kind in kinds}
        res["gemv_bytes"] = e.profile_bytes()
        res["nnz"] = int(torch.count_nonzero(cc).item())
        e.profile(False)
        return res, cc, cc2, tt

    # late: 16 more pulses on the timed engine (the state after the timed run,
    # sparse iterate); early: a fresh engine's pulses warmup..warmup+15 (the
    # dense first pulses of the stream).  The matvec's roofline blends both.
    n_prof = min(args.steps, 16)
    prof, c, c2, t = profiled(eng, idx[args.warmup:args.warmup + n_prof], c, c2, t)
    e2 = Engine(M, n_r, wl.dictionary.ell_idx, wl.dictionary.ell_w, xyz, device=local)
    e2.set_stream(stream)
    if sharded:
        from paper_2603_08582_b200 import sharding

        keep.append(sharding.shard_auto(e2, prefer=args.exchange)[1])
    ce = torch.zeros(M, dtype=torch.float64, device=dev)
    ce2 = torch.empty_like(ce)
    ce, ce2, te = pulse_loop(e2, g_dev, w_dev, d_dev, wl.sigma2, idx[:args.warmup], cfg.steps,
                             cfg.lam_rel, ce, ce2, 1.0, flush)
    prof_early, ce, ce2, te = profiled(e2, idx[args.warmup:args.warmup + n_prof], ce, ce2, te)
    e2.close()
    del ce, ce2
    out["prof"] = prof
    out["prof_early"] = prof_early
    out["n_prof"] = n_prof
    out["shares"] = {k: round(v[1] / n_prof / max(ms / args.steps, 1e-9), 4)
                     for k, v in prof.items() if k in dict(kinds)}
    out["final"] = {"L": eng.scalars()[0], "nnz": int(torch.count_nonzero(c).item()),
                    "last_power_iterations": eng.power_diag()[1]}
    out["eng"] = eng
    out["exchange"] = exch
    out["keep"] = keep
    out["wl"] = wl

    # ---- end-to-end through the public API (host inputs, c_hat read back) ----
    if not args.no_e2e:
        pin_d = torch.from_numpy(np.ascontiguousarray(wl.d)).pin_memory()
        pin_g = torch.from_numpy(np.ascontiguousarray(wl.positions)).pin_memory()
        pin_w = torch.from_numpy(np.ascontiguousarray(wl.omega)).pin_memory()
        stats = api.SufficientStatistics.empty(M, device=local, n_freq=n_r,
                                               dictionary=wl.dictionary, grid=wl.grid)
        if sharded:
            from paper_2603_08582_b200 import sharding

            keep.append(sharding.shard_auto(stats.engine, prefer=args.exchange)[1])
        state = api.SolverState(np.zeros(M), 1.0, stats)
        sc = api.SolverConfig(lam_rel=cfg.lam_rel, inner_steps=cfg.steps)
        cov = api.NoiseCovariance(sigma2=wl.sigma2)
        seen = [0.0]
        pending = collections.deque()

        def drain(keep):
            while len(pending) > keep:
                seen[0] += float(pending.popleft().c_hat[0])  # device -> host read of a result

        def one(k, j, fl):
            # queue pulse k (inputs copied from pinned host memory), then read the
            # result of pulse k - lag: its device->host copy was started when that
            # pulse's FISTA was queued, so it overlaps the pulses queued since
            nonlocal state
            geo = PulseGeometry(j, pin_g[j].numpy(), pin_w.numpy())
            pulse = api.GeometricPulse(pin_d[j].numpy(), geo, cov, wl.grid, wl.dictionary)
            st2 = api.accumulate(state.stats, pulse)
            state = api.online_fista_pulse(
                api.SolverState(state.c_device(local), state.momentum_t, st2), sc)
            if fl is not None:
                fl.fill_(float(k))
            pending.append(state)
            drain(args.e2e_lag)

        for k, j in idx[:args.warmup]:
            one(k, j, flush)
        drain(0)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k, j in idx[args.warmup:]:
            one(k, j, flush)
        drain(0)  # the last results
        e1.record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        e2e_ms = max(e0.elapsed_time(e1), 1e3 * wall)
        if world > 1:
            e2e_ms = max_over_ranks(torch, e2e_ms, dev)
        out["e2e"] = {"value": units * args.steps / (e2e_ms / 1e3), "unit": "pulses/s",
                      "h2d_bytes_per_step": int(3 * 8 + n_r * 8 + n_r * 16),
                      "d2h_bytes_per_step": int(M * 8),
                      "path": "GeometricPulse -> accumulate -> online_fista_pulse -> c_hat (numpy); "
                              f"pulse k's c_hat is read after pulse k+{args.e2e_lag} is queued "
                              "(its device->host copy overlaps those pulses)"
                              + ("; L2 flushed between pulses" if flush is not None else "")}
        del stats, state
    return out


def run_ours(args, rank, world, local):
    import torch

    from paper_2603_08582_b200.workload import CONFIGS
    from dataclasses import replace

    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    base = CONFIGS[args.config]
    sharded = world > 1 and not args.replicas
    cfg = replace(base, seed=base.seed + 1000 * rank) if (rank and not sharded) else base
    clocks = ClockSampler(local)
    clocks.start()
    r = measure_config(args, cfg, rank, world, local, sharded)
    clk = clocks.stop()
    eng, wl = r.pop("eng"), r.pop("wl")
    ms_step = r["ms_per_step"]

    # roofline of the dominant kernel: the FISTA matvec k_gemv_sym streams this
    # rank's share of the packed triangle tile store once per launch
    hbm, bf16, peak_kind = measured_peaks()
    # requested tile bytes / event time over both profiled passes (the
    # support-aware matvec reads only the live slabs / rows of each tile)
    n_gemv = r["prof"]["gemv"][0] + r["prof_early"]["gemv"][0]
    gemv_ms = r["prof"]["gemv"][1] + r["prof_early"]["gemv"][1]
    gemv_bytes = r["prof"]["gemv_bytes"] + r["prof_early"]["gemv_bytes"]
    dense_bytes = eng.n_tiles_local() * 128 * 128 * 4
    bytes_gemv = gemv_bytes / max(n_gemv, 1)
    gemv_avg_ms = gemv_ms / max(n_gemv, 1)
    achieved = bytes_gemv / (gemv_avg_ms * 1e-3) / 1e9

    def regime(p):
        n, t_ms = p["gemv"]
        b = p["gemv_bytes"] / max(n, 1)
        return {"avg_launch_ms": t_ms / max(n, 1), "bytes_per_launch": b,
                "read_fraction_of_store": b / dense_bytes,
                "achieved_gbs": b / (t_ms / max(n, 1) * 1e-3) / 1e9 if n else None,
                "nnz_c": p["nnz"]}
    traffic = None
    prof_json = os.path.join(REPO, "profiles", "ncu_gemv_traffic.json")
    if os.path.exists(prof_json):
        with open(prof_json) as fh:
            tj = json.load(fh)
        if cfg.name in tj and not sharded:
            traffic = tj[cfg.name].get("dram_bytes_per_launch")
    n_gram, gram_ms = r["prof"]["gram"]
    gram_avg = gram_ms / max(n_gram, 1)
    # tensor cores on the default path: K~ = F~ Q F~^H (k_ktc_split / k_ktc_y /
    # k_ktc_z / k_ktc_zsum / k_ktc_assemble, f16x3; the mark spans the five launches)
    n_kt, kt_ms = r["prof"]["ktilde"]
    k_pad = -(-2 * cfg.n_freq // 32) * 32
    kt_flops = 2.0 * wl.dictionary.n_pixels * k_pad * k_pad + 2.0 * q_nnz(wl.dictionary) * k_pad
    kt_avg = kt_ms / max(n_kt, 1)
    kt_tf = kt_flops / (kt_avg * 1e-3) / 1e12 if n_kt else None

    full_arc = None
    if rank == 0 and world == 1 and args.steps < cfg.n_pulses and not args.no_extra:
        # a short run times only the first (dense-iterate) pulses of the stream;
        # the same loop over the whole arc, device-timed, rides along
        import copy

        a2 = copy.copy(args)
        a2.steps, a2.no_e2e = cfg.n_pulses, True
        fa = measure_config(a2, cfg, rank, world, local, False, main=False)
        fa.pop("eng").close()
        fa.pop("wl")
        full_arc = {"value": fa["value"], "ms_per_step": fa["ms_per_step"], "steps": cfg.n_pulses,
                    "warmup": args.warmup,
                    "note": "the same loop over all pulses of the arc (the default `python "
                            "bench.py`): the iterate turns sparse along the arc and the "
                            "support-aware matvec reads less of the store"}
    extra = None
    if rank == 0 and world == 1 and args.config == 3 and not args.no_extra:
        c1 = measure_config(args, CONFIGS[1], rank, world, local, False, main=False)
        e1 = c1.pop("eng")
        c1.pop("wl")
        n1, g1 = c1["prof"]["gemv"]
        extra = {"workload": workload_desc(CONFIGS[1]), "value": c1["value"],
                 "ms_per_step": c1["ms_per_step"], "l2_warm": c1.get("l2_warm"),
                 "e2e": c1.get("e2e"),
                 "gemv": {"avg_launch_ms": g1 / max(n1, 1),
                          "bytes_per_launch": e1.n_tiles * 65536,
                          "note": "34.6 MB store: L2-resident between launches"},
                 "kernel_share_of_step": c1["shares"]}
        e1.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ok, need = oracle_fits(wl.m_atoms)
        if ok:
            v, done, total = cpu_oracle_pulses_per_s(wl, args.cpu_pulses, warm=1)
            cpu = {"value": v, "unit": "pulses/s", "cores": host_cores(), "kind": "port",
                   "sample": f"{done} pulse(s) of {cfg.name} (after 1 untimed) through the "
                             "float64 oracle port of the reference's M-space algorithm, "
                             "numpy/OpenBLAS"}
        else:
            cpu = {"value": None, "unit": "pulses/s", "cores": host_cores(), "kind": "port",
                   "sample": f"not run: needs {need / 1e9:.0f} GB of host RAM"}
    if world > 1:
        torch.distributed.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": r["value"], "unit": "pulses/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak" if args.replicas else "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded, SURVEY App. A); " + (
                "one independent scene per rank" if args.replicas else
                f"one scene, pixel-space state sharded over {world} rank(s)"),
            "config": {
                "workload": workload_desc(cfg),
                "l2": (f"flushed: a {args.flush_l2_mb} MiB buffer (> the 126 MB L2) is written "
                       "between timed pulses, inside the timed region; l2_warm (the same "
                       "pulses unflushed) only where the store fits L2"
                       if args.flush_l2_mb > 0 else "no flush"),
                "mode": eng.mode,
                "precision": "Gram closed form (Dirichlet kernel over the uniform frequency "
                             "grid, fp64-reduced arguments), Re(B) store fp32 packed upper "
                             "triangle, FISTA matvec fp32 (support-aware reads), vectors "
                             "fp64, K~ tcgen05 f16x3",
                "parallelism": (f"replicas x{world}" if args.replicas else
                                f"shard x{world} (tiles of the Re(B) store and K~ pixel tiles "
                                "per rank; y_pix summed over ranks per FISTA step and the K~ "
                                "partials per pulse: " +
                                {"peer": "peer-memory exchange, the slot reduction stores into "
                                         "every rank's device memory (CUDA IPC / NVLink)",
                                 "nccl": "NCCL all-reduce",
                                 "none": "one rank, no exchange"}[r.get("exchange", "none")]
                                + ")"),
                "engine_switches": "none (bench refuses SF_* overrides)",
            },
            "roofline": {"bound": "hbm", "kernel": "k_gemv_sym (FISTA y = Re(B) x, pixel space, "
                                                   "support-aware: live slabs / rows only)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "peak_source": peak_kind, "bytes_per_launch": bytes_gemv,
                         "dense_store_bytes": dense_bytes,
                         "avg_launch_ms": gemv_avg_ms, "launches": n_gemv,
                         "bytes_source": "device counter of the tile bytes each launch requested "
                                         "(sf_profile_bytes), over 16 early pulses of a fresh "
                                         "engine and 16 pulses after the timed run",
                         "early": regime(r["prof_early"]), "late": regime(r["prof"])},
            "gram": {"kernel": "k_gram_dirichlet", "avg_launch_ms": gram_avg,
                     "rmw_bytes_per_launch": 2 * eng.n_tiles_local() * 65536,
                     "achieved_hbm_gbs": 2 * eng.n_tiles_local() * 65536 / (gram_avg * 1e-3) / 1e9,
                     "entries_per_launch": eng.n_tiles_local() * 128 * 128},
            "tensor_core": {
                "gram": "N/A on this path: the default Gram update is the closed form (O(1) "
                        "per stored entry, no contraction); the tensor-core Gram "
                        "(precision='f16x3', atom mode / non-uniform grids) runs at "
                        "sm__pipe_tensor_cycles_active 74.7% at cfg4 "
                        "(profiles/r2_v4_ncu_raw_gram_f16x3_cfg4.csv, 13.3 ms per launch)",
                "kernel": "K~ = F~ Q F~^H on tcgen05 kind::f16, 3 MMAs per product: k_ktc_split "
                          "(fp16 hi/lo slabs) -> k_ktc_y (Y = Q X per Morton tile) -> k_ktc_z "
                          "(split-K Z = X^T Y) -> k_ktc_zsum -> k_ktc_assemble; avg_launch_ms "
                          "spans the five launches inside the pipelined step (ncu of the two "
                          "MMA kernels alone: profiles/README.md)",
                "avg_launch_ms": kt_avg if n_kt else None,
                "algorithmic_flops_per_launch": kt_flops,
                "achieved_tflops": kt_tf,
                "frac_of_bf16_peak": (kt_tf / bf16) if (kt_tf and bf16) else None,
                "bf16_peak_tflops": bf16},
            "kernel_share_of_step": r["shares"], "l2_warm": r.get("l2_warm"),
            "e2e": r.get("e2e"), "gpu_launches": r["gpu_launches"], "clocks": clk,
            "cpu_baseline": cpu, "final": r["final"],
        }
        if full_arc is not None:
            line["full_arc"] = full_arc
        if extra is not None:
            line["cfg1"] = extra
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_batch(args, rank, world, local):
    """BASELINE cfg2: `--scenes` independent cfg0-sized scenes in ONE batched
    engine (every kernel launch covers all scenes).  A step = one pulse for every
    scene; value = scene-pulses/s (one pulse-step of 1024 scenes
    counts as 1024 pulses).  With N ranks the same scenes are split into N
    contiguous slices, one batched engine per rank, no communication (strong
    scaling, BASELINE cfg2 "scene-sharded over 2/4/8 GPUs")."""
    import torch

    from paper_2603_08582_b200 import _lib
    from paper_2603_08582_b200.engine import Engine
    from paper_2603_08582_b200.geometry import pixel_positions
    from paper_2603_08582_b200.workload import CONFIGS, generate_batch
    from dataclasses import replace

    if args.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[2]
    B_total = args.scenes
    lo, hi = B_total * rank // world, B_total * (rank + 1) // world
    scenes = generate_batch(cfg, B_total, device_sim=True)[lo:hi]
    B = hi - lo
    wl = scenes[0]
    M, n_r, P = wl.m_atoms, cfg.n_freq, cfg.n_pulses
    n_total = args.warmup + args.steps
    G = np.ascontiguousarray(np.stack([np.stack([s.positions[k] for s in scenes]) for k in range(P)]))
    D = np.ascontiguousarray(np.stack([np.stack([s.d[k] for s in scenes]) for k in range(P)]))
    S2 = np.ascontiguousarray([s.sigma2 for s in scenes], dtype=np.float64)
    eng = Engine(M, n_r, wl.dictionary.ell_idx, wl.dictionary.ell_w, pixel_positions(wl.grid),
                 device=local, batch=B)
    stream = torch.cuda.current_stream(dev)
    eng.set_stream(stream)
    g_dev, d_dev = torch.from_numpy(G).to(dev), torch.from_numpy(D).to(dev)
    s_dev, w_dev = torch.from_numpy(S2).to(dev), torch.from_numpy(wl.omega).to(dev)
    c = torch.zeros((B, M), dtype=torch.float64, device=dev)
    c2 = torch.empty_like(c)
    flush = (torch.empty(args.flush_l2_mb << 17, dtype=torch.float64, device=dev)
             if args.flush_l2_mb > 0 else None)

    def steps(ks, t, fl):
        nonlocal c, c2
        for k in ks:
            j = k % P
            eng.accumulate_geom_batch(g_dev[j], w_dev, d_dev[j], s_dev)
            t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
            c, c2 = c2, c
            if fl is not None:
                fl.fill_(float(k))
        return t

    t = steps(range(args.warmup), 1.0, flush)
    clocks = ClockSampler(local)
    clocks.start()
    l0 = _lib.launch_count()
    ms, t = timed(torch, stream, world, lambda: steps(range(args.warmup, n_total), t, flush))
    launches = _lib.launch_count() - l0
    clk = clocks.stop()
    value = B_total * args.steps / (ms / 1e3)
    eng.profile(True)
    n_prof = min(args.steps, 4)
    t = steps(range(args.warmup, args.warmup + n_prof), t, flush)
    torch.cuda.synchronize(dev)
    prof = {name: eng.profile_read(kind) for name, kind in
            (("gemv", _lib.K_GEMV), ("gram", _lib.K_GRAM), ("fista_loop", _lib.K_STEP),
             ("operator", _lib.K_OPERATOR), ("fista_call", _lib.K_FISTA))}
    req_bytes = eng.profile_bytes()
    eng.profile(False)
    hbm, _, peak_kind = measured_peaks()
    n_gemv, gemv_ms = prof["gemv"]
    bytes_gemv = req_bytes / max(n_gemv, 1)  # support-aware: requested tile bytes
    gemv_avg = gemv_ms / max(n_gemv, 1)
    achieved = bytes_gemv / (gemv_avg * 1e-3) / 1e9
    shares = {k: round(v[1] / n_prof / max(ms / args.steps, 1e-9), 4) for k, v in prof.items()}

    e2e = None
    if not args.no_e2e:
        pin_g, pin_d = torch.from_numpy(G).pin_memory(), torch.from_numpy(D).pin_memory()
        pin_s, pin_w = torch.from_numpy(S2).pin_memory(), torch.from_numpy(wl.omega).pin_memory()
        host_c = [torch.zeros((B, M), dtype=torch.float64).pin_memory() for _ in range(2)]
        e2 = Engine(M, n_r, wl.dictionary.ell_idx, wl.dictionary.ell_w, pixel_positions(wl.grid),
                    device=local, batch=B)
        te = 1.0

        def host_steps(ks, te):
            for k in ks:
                e2.accumulate_geom_batch(pin_g[k % P].numpy(), pin_w.numpy(), pin_d[k % P].numpy(),
                                         pin_s.numpy())
                te = e2.fista(host_c[k & 1].numpy(), host_c[(k + 1) & 1].numpy(), cfg.steps, te,
                              lam_rel=cfg.lam_rel)  # host c_hat in, host c_hat out (synchronous)
            return te

        te = host_steps(range(args.warmup), te)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        te = host_steps(range(args.warmup, n_total), te)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
        if world > 1:  # the slowest rank's time
            wall = max_over_ranks(torch, wall, dev)
        e2e = {"value": B_total * args.steps / wall, "unit": "pulses/s",
               "h2d_bytes_per_step": int(B * (3 * 8 + n_r * 16 + 8) + n_r * 8 + B * M * 8),
               "d2h_bytes_per_step": int(B * M * 8),
               "path": "Engine.accumulate_geom_batch + Engine.fista on host numpy buffers "
                       "(sf_accumulate_geom_batch / sf_fista, SF_MEM_HOST)"}
        e2.close()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, done, total = cpu_oracle_pulses_per_s(wl, 4, warm=1)
        cpu = {"value": v, "unit": "pulses/s", "cores": host_cores(), "kind": "port",
               "sample": f"{done} pulses of scene 0 of {cfg.name} through the float64 oracle "
                         "port (one scene at a time, as the reference runs), numpy/OpenBLAS"}
    if world > 1:
        torch.distributed.barrier()
    if rank == 0:
        L, n, fb = eng.batch_scalars()
        line = {
            "metric": METRIC, "value": value, "unit": "pulses/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic (seeded, SURVEY App. A; {B_total} scenes, SeedSequence([seed, s]) "
                    "with random azimuth offsets, echoes from the device simulator)",
            "config": {
                "workload": f"{workload_desc(cfg)}; x{B_total} independent scenes, {B} per GPU "
                            "in one batched engine; a step = one pulse for every scene",
                "l2": (f"flushed: a {args.flush_l2_mb} MiB buffer written between timed "
                       "pulse-steps, inside the timed region; " if flush is not None else
                       "no flush: ") + f"{B} pixel-space stores of "
                      f"{eng.n_tiles * 65536 / 1e6:.1f} MB = {B * eng.n_tiles * 65536 / 1e9:.2f} GB "
                      "> 126 MB L2",
                "mode": "pixel", "precision": "Gram closed form, fp32 tile store",
                "parallelism": f"scenes split over {world} rank(s), {B} per rank, no communication",
                "engine_switches": "none (bench refuses SF_* overrides)",
            },
            "roofline": {"bound": "hbm", "kernel": "k_gemv_sym (all scenes' tiles, one launch)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": None, "peak_source": peak_kind,
                         "bytes_per_launch": bytes_gemv, "avg_launch_ms": gemv_avg,
                         "dense_store_bytes": B * eng.n_tiles * 65536,
                         "bytes_source": "device counter of the tile bytes each launch requested "
                                         "(sf_profile_bytes; support-aware warp kernel)",
                         "launches": n_gemv},
            "kernel_share_of_step": shares,
            "e2e": e2e, "gpu_launches": launches, "clocks": clk, "cpu_baseline": cpu,
            "final": {"L_scene0": float(L[0]), "pulses_scene0": int(n[0]),
                      "nnz_scene0": int(torch.count_nonzero(c[0]).item())},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    engine_env_guard()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.config == 2:
        run_batch(args, rank, world, local)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
