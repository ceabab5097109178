O=gpurun_out/r02ad; mkdir -p $O
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline --no-standalone > $O/bench_toy.json 2>> $O/bench.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_lora.json 2>> $O/bench.err
timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_ce.json 2>> $O/bench.err
