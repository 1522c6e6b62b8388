out=gpurun_out/r02d; mkdir -p $out
V=build/variants
bash tools/ab.sh "c2 c3 c5" $V/liblfprobe_b200_LFP_CLS_DIRECT0.so $V/liblfprobe_b200_LFP_CLS_DIRECT1.so 2>&1 | tee $out/ab_cls.txt
LFP_LIB_PATH=$V/liblfprobe_b200_LFP_WAVE_L2_PERSIST1_LFP_WAVE_L2_MISS_NORMAL1.so python tools/c5_steps.py 26 3 2>&1 | tail -1 | tee $out/ab_l2.txt
python tools/diag.py c3 > $out/diag_c3.json 2>&1
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
