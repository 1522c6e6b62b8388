out=gpurun_out/r02p; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2 c5" $V/liblfprobe_b200_LFP_LO_LESS_FAST0_LFP_OCC_PRED0.so $V/liblfprobe_b200_LFP_LO_LESS_FAST1_LFP_OCC_PRED0.so $V/liblfprobe_b200_LFP_LO_LESS_FAST0_LFP_OCC_PRED1.so $V/liblfprobe_b200_LFP_LO_LESS_FAST1_LFP_OCC_PRED1.so 2>&1 | tee $out/ab_lf_pred.txt
python tools/diag.py c3 > $out/diag_c3.json 2>&1
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
