#!/bin/bash
# Debug iteration: GPU parity tests (stop at first failure), trace of the 128^3 ILU(0) sweep, bench k=0,2.
TAG=${1:-d}
shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -15 gpurun_out/pytest_$TAG.log
timeout 300 python tools/trace_psweep.py --nx 128 --k 0 2>&1 | tail -3
for k in 0 2; do
  timeout 300 python bench.py --no-extras --k $k --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_k$k.json 2> gpurun_out/bench_${TAG}_k$k.err
  echo "k=$k: $(python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_k$k.json'));print(round(d['ms_per_step']*1000,1),'us',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
