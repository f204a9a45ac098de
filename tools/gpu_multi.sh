#!/bin/bash
# N>1 bench paths on ONE GPU (ranks share GPU 0): host-staged halo (gloo) and
# the peer transport (CUDA IPC between the processes), for the weak-scaling
# c2 and the strong-scaling c4 workloads.  Numbers are not scaling data (one GPU time-sliced);
# this checks the multi-rank code paths end to end.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
port=29511
for tr in host p2p; do
  for wl in c2 c4; do
    port=$((port + 1))
    SLBM_TRANSPORT=$tr SLBM_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 \
      --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 \
      --workload $wl --steps 6 --warmup 3 --no-cpu > gpurun_out/bench2_${tr}_${wl}.log 2>&1
    echo "bench2 $tr $wl rc=$?"
    tail -1 gpurun_out/bench2_${tr}_${wl}.log | cut -c1-300
  done
done
