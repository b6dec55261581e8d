#!/bin/bash
# Quick GPU iteration: parity tests, then the apply bench for both engines.
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
for k in 0 2; do
  timeout 300 python bench.py --no-extras --k $k --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_k$k.json 2> gpurun_out/bench_${TAG}_k$k.err
  echo "k=$k engine1: $(python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_k$k.json'));print(round(d['ms_per_step']*1000,1),'us',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
  BILUK_ENGINE=0 timeout 300 python bench.py --no-extras --k $k --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_k${k}_e0.json 2> gpurun_out/bench_${TAG}_k${k}_e0.err
  echo "k=$k engine0: $(python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_k${k}_e0.json'));print(round(d['ms_per_step']*1000,1),'us',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
