mkdir -p gpurun_out
export STKDE_BENCH_SHARED_GPU=1
for spec in "social 2" "ornith 4" "stress 8"; do set -- $spec
  echo "== $1 N=$2" >> gpurun_out/reh.log
  timeout 600 python bench.py --gpus $2 --config $1 --steps 5 --warmup 3 >> gpurun_out/reh.log 2>&1; echo rc=$? >> gpurun_out/reh.log
done
