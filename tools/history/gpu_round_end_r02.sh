# r02 round-end pass: GPU suite, smoke, bench lines (default, zerocopy, lora, toy, reference),
# ncu launch list of the default bench command, ncu --set full of one in-pipeline K4 span,
# standalone K3/K4 captures, K4 size sweep.
O=gpurun_out/r02final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_ce.json 2> $O/bench_ce.err
timeout 600 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_zerocopy.json 2> $O/bench_zerocopy.err
timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_scatter_ce.json 2> $O/bench_scatter_ce.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_lora.json 2> $O/bench_lora.err
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_toy.json 2> $O/bench_toy.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 python tools/k4_sizes.py > $O/k4_sizes.jsonl 2> $O/k4_sizes.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_bench_ce.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-standalone > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:materialise_tma -s 0 -c 1 -f \
    -o $O/prof_pipeline_ce python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > $O/ncu_pipeline_ce.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:materialise -c 4 -f \
    -o $O/prof_kernels python tools/ncu_kernels.py > $O/ncu_kernels.log 2>&1
ls -la $O > $O/ls.txt
