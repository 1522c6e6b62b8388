out=gpurun_out/r03e; mkdir -p $out
python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; tail -3 $out/pytest_gpu.log
bash tools/ab.sh "c4 c5 c3" paper_2507_14624_b200/liblfprobe_b200.so 2>&1 | tee $out/ab_default.txt
