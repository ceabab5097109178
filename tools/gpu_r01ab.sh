mkdir -p gpurun_out/streams
for s in 1 2; do
  SLLM_PROFILE_DUMP=1 timeout 600 python bench.py --streams $s --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/streams/bench_ce_s$s.json 2> gpurun_out/streams/bench_ce_s$s.err
  timeout 600 python bench.py --streams $s --steps 5 --warmup 3 --no-cpu-baseline --no-standalone --no-profile > gpurun_out/streams/bench_ce_s${s}_noprof.json 2> gpurun_out/streams/bench_ce_s${s}_noprof.err
done
