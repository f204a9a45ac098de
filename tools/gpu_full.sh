#!/bin/bash
# Round evidence in one gpurun call: gpu_round.sh (smoke, GPU tests, bench,
# ncu launch list + sweep capture), then the other BASELINE configs and the
# C4 strong-scaling workload line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
bash tools/gpu_round.sh
timeout 1500 python tools/bench_configs.py c1 c3 c3h c4 c5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --workload c4 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?" >> gpurun_out/summary.txt
timeout 600 python tools/c4_share.py > gpurun_out/c4_share.jsonl 2> gpurun_out/c4_share.err; echo "c4 share rc=$?" >> gpurun_out/summary.txt
tail -4 gpurun_out/summary.txt
