# compute-sanitizer memcheck over the device parity tests that cover every kernel family
# (TC with TMA, stream / stencil / filter-gradient, tile and block permutes, tap expansion,
# col2im); ~8 min on one B200.  Run on the GPU box:  bash tools/memcheck.sh
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "pairwise or permute_paths or rtr_x_first or execute_golden or backward_random" > gpurun_out/memcheck.txt 2>&1
echo "rc=$?" >> gpurun_out/memcheck.txt
# round 2: plane-conv kernels, strided / 3xTF32 / recompute executors, fused stencils
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_pconv.py tests/test_stride.py \
  tests/test_3xtf32.py tests/test_recompute.py tests/test_fusion.py -x -q -m gpu > gpurun_out/memcheck2.txt 2>&1
echo "rc=$?" >> gpurun_out/memcheck2.txt
tail -3 gpurun_out/memcheck2.txt
tail -3 gpurun_out/memcheck.txt
