TAG=${TAG:-r1_}
mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests/ -x -q -m gpu --durations=15 > gpurun_out/${TAG}pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/${TAG}pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}bench.json 2> gpurun_out/${TAG}bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}bench.json; tail -5 gpurun_out/${TAG}bench.err
