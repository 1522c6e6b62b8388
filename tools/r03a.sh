out=gpurun_out/r03a; mkdir -p $out
V=build/variants
bash tools/ab.sh "c5" $V/liblfprobe_b200_LFP_TFAR0.so $V/liblfprobe_b200_LFP_TFAR1.so 2>&1 | tee $out/ab_tfar.txt
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
