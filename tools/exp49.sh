python tools/prof_permute.py > gpurun_out/perm_new.txt 2>&1
cp paper_2401_03384_b200/libce.so /tmp/new.so; cp paper_2401_03384_b200/libce_old.so paper_2401_03384_b200/libce.so
python tools/prof_permute.py > gpurun_out/perm_old.txt 2>&1
cp /tmp/new.so paper_2401_03384_b200/libce.so
