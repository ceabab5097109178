# r02ae: which ncu --nvtx-include expressions select the verification launches
O=gpurun_out/r02ae; mkdir -p $O
i=0
for x in 'regex:sllm\.verify\..*/' 'regex:.*verify.*/' 'sllm.partition p=0 gpu=0/'; do
  i=$((i+1))
  timeout 300 ncu --metrics gpu__time_duration.sum --nvtx --nvtx-include "$x" -c 2 --csv \
    python bench.py --config toy --steps 1 --warmup 0 --no-cpu-baseline --no-standalone > $O/nvtx_$i.txt 2>&1
  echo "$i [$x] profiled=$(grep -c gpu__time_duration $O/nvtx_$i.txt)" >> $O/summary.txt
done
