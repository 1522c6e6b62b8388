out=gpurun_out/r02s; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2 c5 c4" $V/liblfprobe_b200_LFP_RADII_T1_LFP_UNIFIED0.so $V/liblfprobe_b200_LFP_RADII_T1_LFP_UNIFIED1.so 2>&1 | tee $out/ab_unified.txt
python tools/diag.py c3 > $out/diag_c3.json 2>&1
python tools/diag.py c2 > $out/diag_c2.json 2>&1
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
