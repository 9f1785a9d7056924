"""The peer-memory exchange (sf_peer_*, sharding.shard_peer) across PROCESSES.

Two (and three) processes, one engine each, all on cuda:0: every rank owns its share of
the Re(B) tiles and of the K~ pixel tiles, k_pix_reduce stores the partial
y_pix straight into the rank's slot of BOTH processes' slot arrays (the other
process's array mapped through CUDA IPC -- the same mapping NVLink peers get),
interprocess events order the pushes before the sums, and the hosts meet at a
sequence counter in shared memory.  No kernel waits on another rank's kernel,
so the two ranks can time-slice one GPU (B200_PROFILING.md).  The ranks must
agree bitwise with each other and, to rounding, with an unsharded engine.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import sarfista_oracle as orc
from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2603_08582_b200.dictionary import build_extended_dictionary  # noqa: E402
from paper_2603_08582_b200.engine import Engine  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N_PULSES = 12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_across_processes_matches_unsharded(tmp_path, world):
    port = _free_port()
    outs = [str(tmp_path / f"rank{r}.npz") for r in range(world)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "peer_rank_worker.py"), str(r),
                               str(world), str(port), outs[r], str(N_PULSES)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
             for r in range(world)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=600)[0].decode(errors="replace"))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("peer ranks timed out")
    assert all(p.returncode == 0 for p in procs), "\n".join(logs)
    res = [dict(np.load(o)) for o in outs]
    for r in range(1, world):  # ranks agree bitwise
        assert np.array_equal(res[0]["c"], res[r]["c"]) and res[0]["t"] == res[r]["t"]
        assert np.array_equal(res[0]["L"], res[r]["L"])

    g = {k: v for k, v in golden("oracle_cfg0.npz").items()}
    cfg = CONFIGS[0]
    dic = build_extended_dictionary(cfg.side, cfg.length, cfg.n_rot, cfg.stride)
    m = dic.m_atoms
    dev = torch.device("cuda", 0)
    ref = Engine(m, cfg.n_freq, dic.ell_idx, dic.ell_w, orc.pixel_positions(cfg.side))
    c = torch.zeros(m, dtype=torch.float64, device=dev)
    c2 = torch.empty_like(c)
    t = 1.0
    Ls = []
    for k in range(N_PULSES):
        ref.accumulate_geom(g["positions"][k], g["omega"], g["d"][k], float(g["sigma2"][0]))
        t = ref.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
        c, c2 = c2, c
        Ls.append(ref.scalars()[0])
    ref.close()
    c_ref, L_ref = c.cpu().numpy(), np.array(Ls)
    assert float(res[0]["t"]) == t
    assert rel_l2(res[0]["c"], c_ref) < 1e-5, rel_l2(res[0]["c"], c_ref)
    assert np.max(np.abs(res[0]["L"] - L_ref) / L_ref) < 1e-6


def test_bench_two_ranks_share_one_gpu(tmp_path):
    """bench.py's N > 1 path (launch contract of the driver: torchrun, one rank per
    process) end to end on this one-GPU box: both ranks on cuda:0 with gloo
    (--share-gpu), one scene sharded over them through the peer-memory exchange.
    Only the code path is checked -- the ranks time-slice the GPU."""
    import json

    repo = os.path.dirname(HERE)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(repo, "bench.py"), "--gpus", "2", "--config", "0", "--steps", "6",
           "--warmup", "3", "--share-gpu", "--no-cpu-baseline", "--no-extra"]
    env = {k: v for k, v in os.environ.items() if not k.startswith("SF_")}
    p = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, timeout=600, env=env,
                       cwd=repo)
    assert p.returncode == 0, p.stderr.decode(errors="replace")[-2000:]
    lines = [l for l in p.stdout.decode().splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["steps"] == 6
    assert "peer-memory exchange" in line["config"]["parallelism"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
