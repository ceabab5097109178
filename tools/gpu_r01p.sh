# r01p: bench lines for the remaining BASELINE configs at N=1
mkdir -p gpurun_out
for c in llama2-13b-tp2 llama2-70b-tp8; do for m in ce zerocopy; do
  timeout 600 python bench.py --config $c --mode $m --steps 5 --warmup 3 --cpu-sample-gib 2 > gpurun_out/bench_${c}_$m.json 2> gpurun_out/bench_${c}_$m.err
done; done
timeout 600 python bench.py --config opt-30b --fanout allgather --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2 > gpurun_out/bench_opt30b_allgather.json 2> gpurun_out/bench_opt30b_allgather.err
timeout 900 python bench.py --config llama2-70b --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2 > gpurun_out/bench_llama2-70b-tp1_ce.json 2> gpurun_out/bench_llama2-70b-tp1_ce.err
