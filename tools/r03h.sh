out=gpurun_out/r03h; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2 c5" $V/liblfprobe_b200_LFP_INVK0.so $V/liblfprobe_b200_LFP_INVK1.so 2>&1 | tee $out/ab_invk.txt
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
