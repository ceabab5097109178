# r02ac: worker pool (no thread start / join per load) -- full GPU suite, small-load latency
O=gpurun_out/r02ac; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/host_overhead.py --config toy --reps 50 > $O/host_overhead_toy.jsonl 2>&1
timeout 300 python tools/host_overhead.py --config lora-70b-r32 --reps 20 > $O/host_overhead_lora.jsonl 2>&1
for rep in 1 2; do
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_toy.jsonl 2>> $O/bench.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_lora.jsonl 2>> $O/bench.err
timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
done
