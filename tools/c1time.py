import sys, time, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1509_08360_b200 as pb
from conftest import load_golden, sparse_from
z, _ = load_golden("config1")
S = sparse_from(z)
for dt in ("float64", "float32"):
    dm = pb.DeviceMatrix(S, dt); plan = dm.plan(40)
    for _ in range(5): plan.run(z["coeffs"], 1, omega_kind=pb._lib.OMEGA_SPLITMIX, seed=0)
    dm.ctx.sync()
    t = time.perf_counter(); R = 200
    for _ in range(R): plan.run(z["coeffs"], 1, omega_kind=pb._lib.OMEGA_SPLITMIX, seed=0)
    dm.ctx.sync(); wall = (time.perf_counter() - t) / R * 1e3
    tot, steps, launches = plan.timing()
    print(f"{dt}: wall {wall:.3f} ms/embed, device {tot:.3f} ms, steps {steps:.3f} ms, {launches} K1 launches -> {steps/60*1e3:.1f} us/step")
