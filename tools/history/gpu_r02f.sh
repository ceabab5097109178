O=gpurun_out/r02f; mkdir -p $O
for c in 64 16; do for s in 2 1; do
  echo "=== chunk $c streams $s" >> $O/timeline.txt
  SLLM_PROFILE_DUMP=1 timeout 120 python tools/timeline.py --chunk-mib $c --streams $s 2>> $O/timeline.txt
done; done
