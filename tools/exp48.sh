cat > /tmp/perm1.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2401_03384_b200 as ce
from paper_2401_03384_b200.device import Context, Executor
ctx = Context(0, "auto", graphs=False)
torch.cuda.set_stream(ctx.torch_stream)
for expr in ["bshw->bhws", "bshw->shwb"]:
    plan = ce.optimal(expr, [[128, 256, 14, 14]], "same", "inference")
    ex = Executor(ctx, plan)
    x = ctx.fill_random([128, 256, 14, 14], 1)
    for _ in range(3):
        ex.execute([x])
    torch.cuda.synchronize()
PY
ncu --set full --clock-control none -k regex:transpose --launch-skip 2 --launch-count 1 -o gpurun_out/perm_bhws python /tmp/perm1.py > gpurun_out/ncu_perm.log 2>&1
