timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for k in 0 1 2; do
  timeout 300 python bench.py --no-extras --k $k --steps 20 --warmup 5 > gpurun_out/bench_e_k$k.json 2> gpurun_out/bench_e_k$k.err
  echo "k=$k: $(python -c "import json;d=json.load(open('gpurun_out/bench_e_k$k.json'));print(round(d['ms_per_step']*1000,1),'us',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
