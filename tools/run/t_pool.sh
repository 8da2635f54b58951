PFAC_DEBUG_PLAN=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pool" 2>&1 | tail -5
