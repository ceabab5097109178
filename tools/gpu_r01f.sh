mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/bench_convert.py --config opt-6.7b > gpurun_out/bench_convert.jsonl 2>&1
timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > gpurun_out/bench_scatter_ce.json 2>&1
timeout 600 python bench.py --config lora-70b-r32 --mode ce --steps 20 --warmup 5 --no-cpu-baseline --no-standalone > gpurun_out/bench_lora_ce.json 2>&1
timeout 600 python bench.py --config lora-70b-r32 --mode zerocopy --steps 20 --warmup 5 --no-cpu-baseline --no-standalone > gpurun_out/bench_lora_zc.json 2>&1
