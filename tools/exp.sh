
for k in 0 1 2; do
  timeout 300 python bench.py --no-extras --k $k --steps 20 --warmup 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
  echo "k=$k: $(python -c "import json;d=json.load(open('gpurun_out/bench_c.json'));print(round(d['ms_per_step']*1000,1),'us sweep',round(d['roofline']['kernel_ms']*1000,1))" 2>&1 | tail -1)"
done
