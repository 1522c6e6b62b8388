out=gpurun_out/r03d; mkdir -p $out
V=build/variants
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
bash tools/ab.sh "c2 c4 c1" $V/liblfprobe_b200_LFP_SEG_WW0.so $V/liblfprobe_b200_LFP_SEG_WW1.so 2>&1 | tee $out/ab_ww1.txt
python tools/diag.py c3 > $out/diag_c3.json 2>&1
