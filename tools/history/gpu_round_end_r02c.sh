# r02 final round-end pass (second session): GPU suite, smoke, bench lines, ncu launch list and
# full captures (in-pipeline K4 span, in-pipeline K3 window, standalone K3/K4), sanitizers.
O=${1:-gpurun_out/r02end}
mkdir -p $O/sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_ce.json 2> $O/bench_ce.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_zerocopy.json 2> $O/bench_zerocopy.err
timeout 600 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_scatter_ce.json 2> $O/bench_scatter_ce.err
timeout 300 python bench.py --config lora-70b-r32 --steps 20 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_lora.json 2> $O/bench_lora.err
timeout 300 python bench.py --config toy --steps 50 --warmup 5 --no-cpu-baseline --no-standalone > $O/bench_toy.json 2> $O/bench_toy.err
timeout 600 python bench.py --config llama2-70b-tp8 --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_70b_tp8_p0.json 2> $O/bench_70b_tp8_p0.err
timeout 900 python bench.py --config opt-30b --fanout p2p --steps 3 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_opt30b_p2p.json 2> $O/bench_opt30b_p2p.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_bench_ce.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-standalone > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:materialise_tma -s 0 -c 1 -f \
    -o $O/prof_pipeline_ce python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > $O/ncu_pipeline_ce.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:materialise_tma -s 0 -c 1 -f \
    -o $O/prof_pipeline_scatter_ce python bench.py --mode scatter_ce --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > $O/ncu_pipeline_scatter_ce.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:materialise -c 4 -f \
    -o $O/prof_kernels python tools/ncu_kernels.py > $O/ncu_kernels.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 99 --print-limit 50 python tools/sanitize_gpu.py \
      > $O/sanitizer/$t.log 2>&1; echo "rc=$?" >> $O/sanitizer/$t.log
done
ls -la $O > $O/ls.txt
# 2-rank plumbing on the one GPU (torchrun, gloo): sharded and P2P-fan-out lines
SLLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --config opt-6.7b --steps 3 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_n2_samegpu_none.json 2> $O/bench_n2_samegpu_none.err
SLLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
    bench.py --gpus 2 --config opt-6.7b --fanout p2p --steps 3 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_n2_samegpu_p2p.json 2> $O/bench_n2_samegpu_p2p.err
