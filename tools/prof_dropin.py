import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2109_06976_b200 import dynamics, models
m = models.load("chain7")
for N in (128, 1 << 20):
    rng = np.random.default_rng(1)
    q, qd, u = [rng.uniform(-1, 1, (N, 7)) for _ in range(3)]
    for _ in range(3):
        dynamics.fd_grad(m, q, qd, u)
    t = time.perf_counter(); reps = 20 if N < 1000 else 3
    for _ in range(reps):
        r = dynamics.fd_grad(m, q, qd, u)
    print(N, (time.perf_counter() - t) / reps * 1e6, "us per call")
    pr = cProfile.Profile(); pr.enable()
    for _ in range(reps):
        r = dynamics.fd_grad(m, q, qd, u)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
