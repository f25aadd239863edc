# ncu evidence for profiles/ (round 2: k_sweep).  Each ncu command only after the plain run exits 0.
TAG=${TAG:-r2}
mkdir -p gpurun_out
timeout 600 python tools/ncu_target.py > gpurun_out/${TAG}_target_plain.log 2>&1; echo "plain rc=$?"
# k_raster launches of tools/ncu_target.py: #0 set_mesh's base-mesh count, #1 and #2 full
# evaluations, #3 the cached partial evaluation of colour class 0
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_raster --launch-skip 2 --launch-count 2 \
  -f -o gpurun_out/${TAG}_sweep python tools/ncu_target.py > gpurun_out/${TAG}_ncu_sweep.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out
