# multi-rank plumbing on one GPU (SLLM_BENCH_SAME_GPU=1), multicast probe, LDG zero-copy engine
mkdir -p gpurun_out
python tools/probe_multicast.py > gpurun_out/probe_multicast.json 2>&1
export SLLM_BENCH_SAME_GPU=1
for f in none p2p; do for m in ce zerocopy; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus 2 --steps 3 --warmup 3 --mode $m --fanout $f --no-standalone > gpurun_out/bench_n2same_${f}_${m}.json 2> gpurun_out/bench_n2same_${f}_${m}.err
done; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
     bench.py --gpus 2 --steps 3 --warmup 3 --impl reference > gpurun_out/bench_n2same_reference.json 2> gpurun_out/bench_n2same_reference.err
unset SLLM_BENCH_SAME_GPU
timeout 900 python tools/sweep.py --config opt-6.7b --modes zerocopy,scatter_zc --chunks 64 --streams 2,3 --engines ldg,tma --reps 2 > gpurun_out/sweep_zc_engines.jsonl 2>&1
