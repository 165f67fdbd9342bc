# compute-sanitizer over the paths that changed at the end of round 2: CTA pairs on tt1.0's wide
# 27-stage convs, few-item N tiles on its factor GEMMs, row GEMMs (tests/test_rowgemm.py).
mkdir -p gpurun_out
for L in "tt 1.0" "tk 0.1"; do
  timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/run_layer.py $L 1 > gpurun_out/memcheck_${L// /_}.txt 2>&1
  echo "rc=$?" >> gpurun_out/memcheck_${L// /_}.txt
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_rowgemm.py -x -q -m gpu > gpurun_out/memcheck_rowgemm.txt 2>&1
echo "rc=$?" >> gpurun_out/memcheck_rowgemm.txt
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/run_layer.py tt 1.0 1 > gpurun_out/synccheck_tt10.txt 2>&1
echo "rc=$?" >> gpurun_out/synccheck_tt10.txt
