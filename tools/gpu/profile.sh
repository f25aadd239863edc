# ncu evidence for profiles/ (run under gpurun; each command only after the plain run exits 0)
TAG=${TAG:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/${TAG}_plain.json 2>/dev/null; echo "plain rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "launches rc=$?"
# k_raster launches of tools/ncu_target.py: #0 set_mesh's base-mesh count, #1 and #2
# full evaluations, #3 the cached partial evaluation of colour class 0
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_raster --launch-skip 1 --launch-count 1 \
  -f -o gpurun_out/${TAG}_raster python tools/ncu_target.py > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "full rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_raster --launch-skip 3 --launch-count 1 \
  -f -o gpurun_out/${TAG}_raster_partial python tools/ncu_target.py > gpurun_out/${TAG}_ncu_partial.log 2>&1; echo "partial rc=$?"
# then, here: python tools/summarize_ncu.py r1 gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_raster.ncu-rep gpurun_out/${TAG}_raster_partial.ncu-rep
# (keep the local morea_kernels.cu identical to the profiled build: ncu maps lines to the source on disk)
ls -la gpurun_out
