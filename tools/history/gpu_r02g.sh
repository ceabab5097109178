O=gpurun_out/r02g; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_lora.json 2> $O/bench_lora.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline --streams 1 > $O/bench_lora_s1.json 2> $O/bench_lora_s1.err
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline > $O/bench_toy.json 2> $O/bench_toy.err
timeout 300 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
SLLM_PROFILE_DUMP=1 timeout 120 python tools/timeline.py --chunk-mib 64 --streams 2 2> $O/timeline_lora.txt
