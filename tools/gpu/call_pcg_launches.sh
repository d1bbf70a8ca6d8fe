# C4 512^3 solve launch lists (host PCG loop) and wall times; FL_PCGA selected the PCG order in the round-2 fused-update prototype
for a in 0 1; do
FL_PCGA=$a python tools/profile_solve.py --config c4 --size 512 --host-pcg > gpurun_out/p_plain$a.log 2>&1 && \
FL_PCGA=$a timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/p_launches$a.csv python tools/profile_solve.py --config c4 --size 512 --host-pcg > gpurun_out/p_ncu$a.log 2>&1
done
for a in 0 1 0 1; do FL_PCGA=$a python - >> gpurun_out/p_time$a.txt 2>&1 <<'PY'
import time, torch, sys
sys.path.insert(0, '.')
import paper_2502_04217_b200 as fl
from paper_2502_04217_b200 import workloads
inst = workloads.c4_const(512)
mask = fl.Mask.from_bool(inst.flags, fl.GridShape(inst.dims))
b = fl.observe(torch.from_numpy(inst.beta_true).cuda(), mask)
b += torch.from_numpy(inst.noise).cuda()
for r in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    beta, rep = fl.solve(b, mask, fl.IpmConfig(lam=inst.lam))
    torch.cuda.synchronize(); print(r, time.perf_counter() - t, rep.krylov_counts, flush=True)
PY
done
