# r02y: L2 evict-first hints on the ring's bulk loads / the tensor stores (A/B builds)
O=gpurun_out/r02y; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for rep in 1 2; do
for v in default ldhint sthint bothhint; do
  if [ $v = default ]; then unset SLLM_LIB_PATH; else export SLLM_LIB_PATH=build/ab/$v/libsllm.so; fi
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:materialise -c 4 python tools/ncu_kernels.py 2>/dev/null \
     | grep materialise | sed "s/^/$v,$rep,/" >> $O/ncu_variants.csv
  timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/bench_ce.jsonl 2>> $O/bench.err
  timeout 300 python bench.py --mode scatter_ce --steps 5 --warmup 3 --no-cpu-baseline --no-standalone | sed "s/^{/{\"variant\": \"$v\", \"rep\": $rep, /" >> $O/bench_scatter.jsonl 2>> $O/bench.err
done; done
unset SLLM_LIB_PATH
