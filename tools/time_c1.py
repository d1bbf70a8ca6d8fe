import cProfile, pstats, sys, time, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tests")
import numpy as np, torch
import paper_2502_04217_b200 as fl
from paper_2502_04217_b200 import workloads
from conftest import load_golden
g = load_golden("solve_c1_4096")
dims = tuple(int(d) for d in g["dims"])
mask = fl.Mask(g["missing"], fl.GridShape(dims))
b = torch.from_numpy(g["b"]).cuda()
cfg = fl.IpmConfig(lam=float(g["lam"]))
for _ in range(5): fl.solve(b, mask, cfg)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): fl.solve(b, mask, cfg)
torch.cuda.synchronize()
print("solve ms", (time.perf_counter() - t) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): fl.solve(b, mask, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
