#!/bin/bash
# Multi-GPU bench lines on one box: tools/run_multi.sh <tag> "<bench args>" [N ...]
# writes gpurun_out/<tag>_n<N>.json / .err per GPU count (each run bounded by timeout).
tag=$1; shift
args=$1; shift
port=29611
for n in "$@"; do
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py $args > gpurun_out/${tag}_n1.json 2> gpurun_out/${tag}_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $n $args > gpurun_out/${tag}_n${n}.json 2> gpurun_out/${tag}_n${n}.err
  fi
  echo "== $tag n=$n rc=$?"
  tail -c 200 gpurun_out/${tag}_n${n}.json; echo
  port=$((port + 1))
done
