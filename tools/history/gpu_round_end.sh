# r01y: round-end pass -- GPU suite, smoke, bench lines, ncu launch list + full captures
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench_ce.json 2> $O/bench_ce.err
timeout 600 python bench.py --mode zerocopy --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_zerocopy.json 2> $O/bench_zerocopy.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-standalone > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:materialise -c 4 -f \
    -o $O/prof_kernels python tools/ncu_kernels.py > $O/ncu_kernels.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:materialise_tma -s 2 -c 1 -f \
    -o $O/prof_pipeline_ce python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > $O/ncu_pipeline_ce.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:materialise_tma -s 1 -c 1 -f \
    -o $O/prof_pipeline_scatter_ce python bench.py --mode scatter_ce --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > $O/ncu_pipeline_scatter_ce.log 2>&1

# 2 ranks on the one GPU (gloo plumbing of the multi-rank paths; numbers share one PCIe link)
for f in none p2p; do
  SLLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --fanout $f --no-standalone --cpu-sample-gib 1 \
      > $O/bench_n2_samegpu_$f.json 2> $O/bench_n2_samegpu_$f.err
done

ls -la $O > $O/ls.txt
