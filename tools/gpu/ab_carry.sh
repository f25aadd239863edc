mkdir -p gpurun_out
MOREA_LIB=$PWD/build/var/carry.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_next4.py tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/carry_pytest.log 2>&1; echo "carry pytest rc=$?"; tail -3 gpurun_out/carry_pytest.log
AB_ROUNDS=3 timeout 900 python tools/ab.py build/var/base.so build/var/carry.so > gpurun_out/ab_carry.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_carry.log
