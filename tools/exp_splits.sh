for sp in 9,16 1,128 2,64 4,32 8,16 12,12; do
  BILUK_SPLIT=$sp timeout 300 python bench.py --no-extras --k 0 --steps 20 --warmup 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
  echo "split $sp: $(python -c "import json;d=json.load(open('gpurun_out/bench_c.json'));print(round(d['ms_per_step']*1000,1),'us sweep',round(d['roofline']['kernel_ms']*1000,1))" 2>&1 | tail -1)"
done
BILUK_SPLIT=1,128 python tools/trace_psweep.py --k 0 --out gpurun_out/ptrace_z.npz > gpurun_out/trz.log 2>&1
