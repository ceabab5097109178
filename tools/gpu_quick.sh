# quick check: GPU tests + CE bench (+ NCU=1: in-pipeline ncu capture of a K4 verification launch + launch list)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for m in ${BENCH_MODES:-ce}; do
  timeout 600 python bench.py --mode $m --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err
done
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:materialise_tma -s 2 -c 1 -f \
      -o gpurun_out/prof_pipeline_ce python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > gpurun_out/ncu_pipeline.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-standalone > gpurun_out/ncu_bench.log 2>&1
fi
