# Round-end evidence: the default bench (CPU legs included), then the ncu launch
# list of the bench command and one --set full capture of k_raster's full and
# cached partial launches (each ncu command only after its plain run exits 0).
TAG=${TAG:-r2}
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/${TAG}_plain.json 2>/dev/null; echo "plain rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "launches rc=$?"
timeout 600 python tools/ncu_target.py > gpurun_out/${TAG}_target_plain.log 2>&1; echo "target rc=$?"
# k_raster launches of tools/ncu_target.py: #0 set_mesh's base-mesh count, #1 and #2
# full evaluations, #3 the cached partial evaluation of colour class 0
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_raster --launch-skip 2 --launch-count 2 \
  -f -o gpurun_out/${TAG}_raster python tools/ncu_target.py > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out
