O=gpurun_out/r02aj; mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_ce.json 2> $O/bench_ce.err
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline --no-standalone > $O/bench_toy.json 2> $O/bench_toy.err
