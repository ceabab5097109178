# Every BASELINE config at N=1 on the final code, one box, one JSON line each -> gpurun_out/all/bench_all.jsonl
mkdir -p gpurun_out/all
O=gpurun_out/all/bench_all.jsonl; : > $O
run() { timeout 900 python bench.py "$@" 2>> gpurun_out/all/bench_all.err | tail -1 >> $O; }
run --config toy --steps 20 --warmup 5 --no-standalone --cpu-sample-gib 1
for m in ce zerocopy scatter_ce scatter_zc; do run --config opt-6.7b --mode $m --steps 5 --warmup 3; done
run --config llama2-13b-tp2 --steps 5 --warmup 3 --cpu-sample-gib 2
run --config llama2-13b-tp2 --all-partitions --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2
run --config llama2-70b-tp8 --steps 5 --warmup 3 --cpu-sample-gib 2
run --config llama2-70b-tp8 --all-partitions --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2
run --config llama2-70b --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2
for f in none p2p bcast allgather; do run --config opt-30b --fanout $f --steps 3 --warmup 3 --no-standalone --cpu-sample-gib 2; done
run --config lora-70b-r32 --steps 20 --warmup 5 --no-standalone --cpu-sample-gib 1
