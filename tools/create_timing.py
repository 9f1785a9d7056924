"""Host cost of engine creation and of small dense accumulate calls (the
reference-API scale of the acceptance criteria: M <= 32, N_r <= 16)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2603_08582_b200 import solver as sf  # noqa: E402
from paper_2603_08582_b200.engine import Engine  # noqa: E402

t0 = time.perf_counter()
e = Engine(8, 4, keep_complex=True)
print(f"first engine (context init) {1e3 * (time.perf_counter() - t0):.1f} ms")
e.close()
for kc in (False, True):
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        e = Engine(20, 12, keep_complex=kc)
        ts.append(time.perf_counter() - t0)
        e.close()
    print(f"Engine(20, 12, keep_complex={kc}) median {1e3 * np.median(ts):.2f} ms")
rng = np.random.default_rng(0)
G = rng.standard_normal((12, 20)) + 1j * rng.standard_normal((12, 20))
d = rng.standard_normal(12) + 1j * rng.standard_normal(12)
stats = sf.SufficientStatistics.empty(20)
p = sf.PulseMeasurement(d, G, sf.NoiseCovariance(sigma2=1.0))
stats = sf.accumulate(stats, p)
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    stats = sf.accumulate(stats, p)
    ts.append(time.perf_counter() - t0)
print(f"accumulate (dense, M=20) median {1e3 * np.median(ts):.3f} ms")
ts = []
for _ in range(20):
    t0 = time.perf_counter()
    A = stats.A
    ts.append(time.perf_counter() - t0)
print(f"stats.A median {1e3 * np.median(ts):.3f} ms")
t0 = time.perf_counter()
for seed in range(20):
    s = sf.SufficientStatistics.empty(20)
    for _ in range(5):
        s = sf.accumulate(s, p)
    _ = s.A, s.b
print(f"20 x (empty + 5 accumulate + A, b): {1e3 * (time.perf_counter() - t0):.1f} ms")
