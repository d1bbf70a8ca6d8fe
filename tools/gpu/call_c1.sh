# C1 latency breakdown: solve wall time (graph / host PCG loop), per-piece device times, launch list
timeout 300 python tools/c1_latency.py > gpurun_out/c1_latency.json 2> gpurun_out/c1_latency.err; echo "rc=$?" >> gpurun_out/c1_latency.err
