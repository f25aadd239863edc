#!/bin/bash
# GPU-box helper: parity tests, then a short bench (no CPU leg, no extras).
TAG=${TAG:-r2_}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests/ -q -m gpu ${PYTEST_ARGS} --durations=10 > gpurun_out/${TAG}pytest.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/${TAG}pytest.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:---no-extras} > gpurun_out/${TAG}bench.json 2> gpurun_out/${TAG}bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}bench.json; tail -5 gpurun_out/${TAG}bench.err
fi
