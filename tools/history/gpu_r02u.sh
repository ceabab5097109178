# r02u: zero-copy host reads with the L2 256-byte fill hint (LDG engine) vs without; TMA ref
O=gpurun_out/r02u; mkdir -p $O
for rep in 1 2; do
timeout 300 python bench.py --mode zerocopy --engine ldg --steps 5 --warmup 2 --no-cpu-baseline --no-standalone | sed "s/^{/{\"variant\": \"ldg\", /" >> $O/zc_l2.jsonl 2>> $O/zc.err
SLLM_LIB_PATH=build/ab/l2pf256/libsllm.so timeout 300 python bench.py --mode zerocopy --engine ldg --steps 5 --warmup 2 --no-cpu-baseline --no-standalone | sed "s/^{/{\"variant\": \"ldg_l2_256B\", /" >> $O/zc_l2.jsonl 2>> $O/zc.err
timeout 300 python bench.py --mode zerocopy --steps 5 --warmup 2 --no-cpu-baseline --no-standalone | sed "s/^{/{\"variant\": \"tma\", /" >> $O/zc_l2.jsonl 2>> $O/zc.err
done
