out=gpurun_out/r02z; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2 c5 c4" $V/liblfprobe_b200_LFP_HI_REORDER0.so $V/liblfprobe_b200_LFP_HI_REORDER1.so 2>&1 | tee $out/ab_reorder.txt
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
