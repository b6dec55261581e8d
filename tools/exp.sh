# ad-hoc A/B on the 128^3 sweep (bench.py --no-extras); exp_lib/<variant>/libbiluk.so builds via BILUK_LIB_PATH
run() {  # label, k, env...
  local label=$1 k=$2; shift 2
  env "$@" timeout 300 python bench.py --no-extras --k $k --steps 20 --warmup 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
  echo "$label k=$k: $(python -c "import json;d=json.load(open('gpurun_out/bench_c.json'));print(round(d['ms_per_step']*1000,1),'us sweep',round(d['roofline']['kernel_ms']*1000,1))" 2>&1 | tail -1)"
}
for k in ${KS:-0 2}; do
  for v in ${VARIANTS:-}; do run $v $k BILUK_LIB_PATH=$PWD/exp_lib/$v/libbiluk.so; done
  for e in ${ENVS:-}; do run $e $k $(echo $e | tr '+' ' '); done
done
