#!/bin/bash
# Fast GPU iteration: a small parity subset, the trace, the k=0 and k=2 apply bench.
TAG=${1:-it}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "synthetic or deterministic" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
timeout 120 python tools/trace_psweep.py --nx 128 --k 0 --out gpurun_out/ptrace_$TAG.npz 2>&1 | tail -1
for k in 0 2; do
  timeout 150 python bench.py --no-extras --k $k --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_k$k.json 2> gpurun_out/bench_${TAG}_k$k.err
  echo "k=$k: $(python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_k$k.json'));print(round(d['ms_per_step']*1000,1),'us',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
