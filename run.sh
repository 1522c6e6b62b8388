python -m pytest tests/test_pointbake.py -x -q -k "at_scale" 2>&1 | grep -E "^E " | head -20 > gpurun_out/pb_tests.log
