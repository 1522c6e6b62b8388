out=gpurun_out/r03i; mkdir -p $out
V=build/variants
bash tools/ab.sh "c3 c2 c5 c4" $V/liblfprobe_b200_LFP_FK0.so $V/liblfprobe_b200_LFP_FK1.so 2>&1 | tee $out/ab_fk.txt
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
