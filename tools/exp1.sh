for L in "tk 0.1" "tk 1.0" "tt 0.1" "tt 1.0"; do TAG="$L" python tools/tc_timing.py $L; done > gpurun_out/timing.txt 2>&1
python tools/tc_phases.py >> gpurun_out/timing.txt 2>&1
EXTRA_DBG=1 python tools/tc_phases.py >> gpurun_out/timing.txt 2>&1
EXTRA_DBG=4 python tools/tc_phases.py >> gpurun_out/timing.txt 2>&1
