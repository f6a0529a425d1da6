# tensor-core block sweep: accuracy, block tests, throughput probes
timeout 60 python scripts/tc_err.py
timeout 300 python -m pytest tests/test_gpu_block_large.py tests/test_gpu_block.py -q -x 2>&1 | tail -4
timeout 120 python scripts/tc_dots_probe.py 0 16
