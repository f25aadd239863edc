# dev loop on the GPU box: quick parity subset + bench (no oracle leg, no extras)
TAG=${TAG:-dev_}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_sobol.py -x -q -m gpu ${PYTEST_EXTRA} > gpurun_out/${TAG}pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/${TAG}pytest.log
timeout 900 python bench.py --no-cpu-baseline --no-extras ${BENCH_EXTRA} > gpurun_out/${TAG}bench.json 2> gpurun_out/${TAG}bench.err; echo "bench rc=$?"
python - <<'PY'
import json,os
t=os.environ.get("TAG","dev_")
try:
    d=json.load(open(f"gpurun_out/{t}bench.json"))
    b=d["breakdown"]
    print("value",round(d["value"]),"full_ms",round(b["full_ms"],2),"partial_ms",round(b["partial_ms"],2),"frac",round(d["roofline"]["frac"],4),"clk",d["clocks"])
except Exception as e:
    print("bench parse failed", e)
PY
tail -3 gpurun_out/${TAG}bench.err
