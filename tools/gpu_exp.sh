#!/bin/bash
# Ad-hoc GPU experiment runner: executes the commands in $EXP (one per line),
# each under a timeout, logging to gpurun_out/exp_<k>.log.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
k=0
while IFS= read -r cmd; do
  [ -z "$cmd" ] && continue
  k=$((k+1))
  echo "== $cmd" > gpurun_out/exp_$k.log
  timeout ${EXP_TIMEOUT:-600} bash -c "$cmd" >> gpurun_out/exp_$k.log 2>&1
  echo "rc=$?" >> gpurun_out/exp_$k.log
  tail -4 gpurun_out/exp_$k.log
done <<< "$EXP"
