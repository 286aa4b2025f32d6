#!/bin/bash
# GPU box: host facts, then the GPU test suite (optionally a subset: $@ passed to pytest)
mkdir -p gpurun_out
{ nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; free -g | head -2; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; } > gpurun_out/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest -q -m gpu -x "${@:-tests}" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
