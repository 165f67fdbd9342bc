# ncu --set full of one launch per SIMT / permute / fused kernel family (SURVEY §8 D2/D3:
# achieved HBM GB/s for the memory-bound families), on the CP ResNet-34 conv2_x layer
# (64->64 @56, B=128) at cr 1.0 (R=275: stencil + dwgrad) and cr 0.1 (R=27: fused dw2).
NCU="ncu --set full --import-source on --clock-control none --launch-count 1"
L1="tools/run_layer.py cp 1.0 1 64 64 3 56 128"
L2="tools/run_layer.py cp 0.1 1 64 64 3 56 128"
timeout 600 $NCU -k regex:ce_dw_kernel -o gpurun_out/full_cp10_stencil python $L1 > gpurun_out/ncuf1.log 2>&1
timeout 600 $NCU -k regex:ce_dwgrad_kernel -o gpurun_out/full_cp10_dwgrad python $L1 > gpurun_out/ncuf2.log 2>&1
timeout 600 $NCU -k regex:ce_dw2_kernel -o gpurun_out/full_cp01_dw2 python $L2 > gpurun_out/ncuf3.log 2>&1
timeout 600 $NCU -k regex:ce_transpose -o gpurun_out/full_tk10_permute python tools/run_layer.py tk 1.0 1 > gpurun_out/ncuf4.log 2>&1
timeout 600 $NCU -k regex:ce_stream -o gpurun_out/full_cp_conv1_stream python tools/run_layer.py cp 1.0 1 64 3 7 112 32 > gpurun_out/ncuf5.log 2>&1
# plane-conv kernels (ce_pconv.cu) on cfg3's RTR conv1 (B=256): forward and filter gradient
L3="tools/prof_layer.py rtr 4,4,4 1,1,3 7 112 256 0.1"
timeout 600 $NCU -k regex:ce_pconv_kernel -o gpurun_out/full_rtr_conv1_pconv python $L3 > gpurun_out/ncuf6.log 2>&1
timeout 600 $NCU -k regex:ce_pconv_wgrad -o gpurun_out/full_rtr_conv1_pconv_wgrad python $L3 > gpurun_out/ncuf7.log 2>&1
