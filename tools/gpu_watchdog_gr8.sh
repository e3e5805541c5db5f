MTKV_NVCC_EXTRA="-DMTKV_WATCHDOG" python -m paper_2604_22881_b200.build --force > /dev/null 2>&1 || echo build failed
MTKV_GEMM_WIDE=256 timeout 120 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -s -k "gr8" > gpurun_out/wd3.log 2>&1
grep -c watchdog gpurun_out/wd3.log; grep watchdog gpurun_out/wd3.log | head -8; tail -3 gpurun_out/wd3.log
