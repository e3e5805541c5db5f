timeout 300 python -m pytest tests/test_gpu_engine.py -q -m gpu -x -s -k "attention" 2>&1 | grep -E "passed|failed|Error|assert|Timeout" > gpurun_out/p13_gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 4 --no-cpu-baseline > gpurun_out/p13_bench.log 2>&1
MTKV_ATTN_TRACE=gpurun_out/attn_trace13.bin timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/trace13_bench.log 2>&1; python tools/attn_trace.py gpurun_out/attn_trace13.bin 4 > gpurun_out/attn_trace13.txt 2>&1
