# ILU(0) sweep time over (y, z) part splits (BILUK_SPLIT diagnostics)
for sp in ${SPLITS:-9,16 11,13 8,18 13,11 10,14}; do
  BILUK_SPLIT=$sp timeout 300 python bench.py --no-extras --k 0 --steps 20 --warmup 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
  echo "split $sp: $(python -c "import json;d=json.load(open('gpurun_out/bench_c.json'));print(round(d['ms_per_step']*1000,1),'us sweep',round(d['roofline']['kernel_ms']*1000,1))" 2>&1 | tail -1)"
done
