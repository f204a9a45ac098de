#!/bin/bash
# N>1 bench path on ONE GPU: two ranks share GPU 0, halo over host memory + gloo.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
SLBM_TRANSPORT=host SLBM_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 > gpurun_out/bench2.log 2>&1
echo "bench2 rc=$?"
tail -1 gpurun_out/bench2.log
