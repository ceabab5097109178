O=gpurun_out/r02ar; mkdir -p $O
SLLM_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29537 \
    bench.py --gpus 2 --config opt-6.7b --fanout p2p --steps 3 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_n2_p2p.json 2> $O/bench_n2_p2p.err
timeout 900 python bench.py --config opt-30b --fanout bcast --steps 3 --warmup 3 --no-cpu-baseline --no-standalone > $O/bench_opt30b_bcast.json 2> $O/bench_opt30b_bcast.err
