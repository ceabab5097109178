# r02 round-end pass (third session: in-process peer groups ordered by CUDA events; no multi-process P2P on one GPU):
# GPU suite, smoke, bench lines, ncu launch list and full captures (in-pipeline K4 span, in-pipeline K3 window,
# standalone K3/K4), in-process P2P groups on the one GPU, multi-rank sharded plumbing.
O=${1:-gpurun_out/r02end}
mkdir -p $O
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
# (compute-sanitizer is closed on the GPU pool from this session on; earlier clean logs: profiles/r02/final4/sanitizer)
timeout 600 python tools/probe_p2p_group.py > $O/probe_p2p_group.log 2>&1; echo rc=$? >> $O/probe_p2p_group.log
ls -la $O > $O/ls.txt
# 2-rank plumbing on the one GPU (torchrun, gloo): sharded and P2P-fan-out lines (the P2P ranks wait for each
# other's flags on the host: SLLM_PEER_WAIT=host, set by bench.py under SLLM_BENCH_SAME_GPU)
SLLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --config opt-6.7b --steps 3 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_n2_samegpu_none.json 2> $O/bench_n2_samegpu_none.err
SLLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
    bench.py --gpus 2 --config opt-6.7b --fanout p2p --steps 3 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_n2_samegpu_p2p.json 2> $O/bench_n2_samegpu_p2p.err
# 4 and 8 ranks on the one GPU (plumbing of the N > 1 bench path: barriers, B_h2d(N), max over ranks)
SLLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 \
    bench.py --gpus 4 --config opt-6.7b --steps 2 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_n4_samegpu_none.json 2> $O/bench_n4_samegpu_none.err
SLLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29536 \
    bench.py --gpus 8 --config toy --steps 5 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_n8_samegpu_toy.json 2> $O/bench_n8_samegpu_toy.err
# K3 standalone on the LLaMA-2-70B TP8 rank-0 layout
NCU_CONFIG=llama2-70b-tp8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:materialise -c 4 -f \
    -o $O/prof_kernels_70b_tp8 python tools/ncu_kernels.py > $O/ncu_kernels_70b_tp8.log 2>&1
