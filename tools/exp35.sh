{
for m in auto fp32; do MATH=$m TAG=$m timeout 120 python tools/tc_timing.py tt 1.0; MATH=$m TAG=$m timeout 120 python tools/tc_timing.py tk 0.1; done
} > gpurun_out/exp35.txt 2>&1
