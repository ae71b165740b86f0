#!/usr/bin/env bash
# Dry runs of `bench.py --gpus N` on a one-GPU box: N ranks time-slicing cuda:0
# over gloo (PWADV_BENCH_SHARE_GPU=1) — the N>1 control path (CUDA IPC mapping,
# flag handshake, per-rank self-checks, agreed fallbacks, JSON line), not a
# measurement. One line per run into gpurun_out/dry/lines.jsonl.
#   /usr/local/graft/bin/gpurun --timeout 1500 -- bash tools/dry_run_multi.sh
set -u
OUT=gpurun_out/dry; mkdir -p $OUT; : > $OUT/lines.jsonl
export PWADV_BENCH_SHARE_GPU=1
run() {  # run N CONFIG [extra args]
  local n=$1 cfg=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 2000)) bench.py --gpus $n --config $cfg --steps 10 --warmup 3 --no-cpu "$@" \
    > $OUT/n${n}_$cfg.out 2> $OUT/n${n}_$cfg.err
  echo "n=$n $cfg rc=$?"
  grep '^{' $OUT/n${n}_$cfg.out >> $OUT/lines.jsonl
  grep -h "^bench:" $OUT/n${n}_$cfg.err | sort | uniq -c
}
run 2 c1
run 4 c1
run 8 c1
run 2 c2
run 8 c2
run 2 c3 --no-e2e
run 2 c4
run 4 c4 --no-e2e
