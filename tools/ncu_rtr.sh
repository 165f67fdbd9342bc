set -x
L='python tools/prof_layer.py rtr 4,4,8 4,4,4 3 28 256 0.1'
for k in ce_stream_blk ce_stream_klane "ce_stream_kernel" ce_rowcopy ; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -c 1 -o gpurun_out/rtr28_$k $L > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:transpose64 -s 1 -c 1 -o gpurun_out/rtr28_transpose64 $L > /dev/null 2>&1
ls -la gpurun_out/
