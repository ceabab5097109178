# r02b: GPU suite after the hardening / NCCL-unit / bench changes, then bench lines
O=gpurun_out/r02b
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for f in bcast allgather; do
  timeout 600 python bench.py --fanout $f --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_opt30b_$f.json 2> $O/bench_opt30b_$f.err
done
SLLM_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --config opt-6.7b --fanout p2p --steps 3 --warmup 2 \
   > $O/bench_n2_samegpu_p2p.json 2> $O/bench_n2_samegpu_p2p.err
timeout 300 python bench.py --gpus 2 --steps 1 --warmup 1 > $O/bench_gpus2_on_1gpu.json 2> $O/bench_gpus2_on_1gpu.err; echo "rc=$?" >> $O/bench_gpus2_on_1gpu.err
