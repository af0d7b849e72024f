import sys, json; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2109_06976_b200 import models
from paper_2109_06976_b200.rollout import Rollout
for robot, B, H in (("chain7", 128, 64), ("chain7", 4096, 64), ("quad12", 128, 64), ("humanoid30", 128, 32)):
    m = models.load(robot); n = m.n_dof
    rng = np.random.default_rng(1)
    q0 = torch.from_numpy(rng.uniform(-1, 1, (B, n))).cuda(); tau = torch.from_numpy(rng.uniform(-1, 1, (B, H, n))).cuda()
    for fused in (True, False):
        r = Rollout(m, B, H, 0.01, "f64", grad=True, graph=True, fused=fused)
        for _ in range(3): r.run(q0, q0, tau)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): r.run(q0, q0, tau)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps({"robot": robot, "B": B, "H": H, "fused": fused, "us": e0.elapsed_time(e1) / 10 * 1e3}))
