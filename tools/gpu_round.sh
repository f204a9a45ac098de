#!/bin/bash
# One gpurun call: smoke, GPU tests, bench, ncu launch list of the bench command
# + one full capture of the two AA sweep kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/summary.txt
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
if [ -z "$NO_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
fi
timeout 600 python bench.py ${BENCH_ARGS:---steps 200 --warmup 10} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu --sustained-s 0 > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_index_sweep|k_aa_odd" -s 2 -c 2 -o gpurun_out/prof_aa -f python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/summary.txt
fi
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt 2>/dev/null
tail -1 gpurun_out/bench.log >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
