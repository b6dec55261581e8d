#!/bin/bash
# One gpurun call: GPU tests, smoke, the bench line, the ncu launch list and one full capture of the sweep.
#   gpurun --timeout 3000 -- bash tools/gpu_round.sh [tag]
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1; lscpu > gpurun_out/lscpu_$TAG.txt 2>&1
timeout 1700 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 4 --warmup 3 --no-extras > gpurun_out/launches_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psweep_kernel -s 3 -c 1 -f -o gpurun_out/sweep_$TAG \
    python tools/profile_sweep.py --nx 128 --k 0 --spmv 0 > gpurun_out/ncu_sweep_$TAG.log 2>&1
echo done
