./oracle/_ref/reftests 2>&1 | tail -30
timeout 900 python -m pytest -q -x tests/test_gpu_reftests.py tests/test_gpu_dropin.py tests/test_gpu_parity.py 2>&1 | grep -E "FAIL|Error|assert|passed|failed" | head -20
