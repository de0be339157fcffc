#!/bin/bash
# One GPU-box pass: tests, smoke, bench, ncu launch list + full capture of the top kernel.
# usage (via gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel|eval_kernel" -s 3 -c 1 \
    -o gpurun_out/${TAG}_prof python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done eval
# Newton solve (f1) capture of the same build
timeout 900 ncu --set full --clock-control none --import-source on -k regex:newton_kernel -s 1 -c 1 \
    -o gpurun_out/${TAG}_newton_prof python tools/newton_prof.py > gpurun_out/${TAG}_newton_ncu.log 2>&1
echo done newton
