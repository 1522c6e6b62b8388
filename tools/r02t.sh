out=gpurun_out/r02t; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2 c5 c4" $V/liblfprobe_b200_LFP_TFORM0.so $V/liblfprobe_b200_LFP_TFORM1.so 2>&1 | tee $out/ab_tform.txt
bash tools/ab.sh "c3 c2" $V/liblfprobe_b200_LFP_MIN_BLOCKS5.so 2>&1 | tee -a $out/ab_tform.txt
bash tools/ab.sh "c5" $V/liblfprobe_b200_LFP_WAVE_MIN_BLOCKS8.so $V/liblfprobe_b200_LFP_WAVE_CF_SMEM0.so 2>&1 | tee -a $out/ab_tform.txt
python tools/diag.py c3 > $out/diag_c3.json 2>&1
python tools/diag.py c2 > $out/diag_c2.json 2>&1
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
