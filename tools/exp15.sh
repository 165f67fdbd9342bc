timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/exp15.txt
echo "rc=$?" >> gpurun_out/exp15.txt
