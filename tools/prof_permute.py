"""Time unary permute plans (family c) in isolation: python tools/prof_permute.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_03384_b200 as ce  # noqa: E402
from paper_2401_03384_b200.device import Context, Executor  # noqa: E402

CASES = [
    ("bshw->bhws", [[128, 256, 14, 14]]),
    ("bshw->shwb", [[128, 256, 14, 14]]),
    ("bhwr->rbhw", [[128, 14, 14, 229]]),
    ("abcdef->dabcef", [[256, 4, 4, 4, 28, 28]]),
    ("abcdhwxy->bcdhwxya", [[256, 4, 4, 4, 28, 28, 10, 10]]),
    ("abcdhwxy->yabcdhwx", [[64, 4, 4, 4, 28, 28, 10, 10]]),
    ("bthw->btwh", [[128, 256, 14, 14]]),
    ("abcde->eabcd", [[256, 3136, 10, 10, 4]]),        # RTR pack: 4-wide in, 10-wide out
    ("abcdef->abdcfe", [[256, 784, 4, 16, 10, 10]]),  # 10x10 transposes under a batch
    ("ab->ba", [[3211264, 4]]),                        # 4-wide output unit axis
]
ctx = Context(0, "auto")
torch.cuda.set_stream(ctx.torch_stream)
for expr, dims in CASES:
    plan = ce.optimal(expr, dims, "same", "inference")
    ex = Executor(ctx, plan)
    x = ctx.fill_random(dims[0], 1)
    for _ in range(3):
        ex.execute([x])
    torch.cuda.synchronize()
    st = ctx.torch_stream
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ex.execute([x])
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms_call = sorted(ts)[len(ts) // 2]
    ex.set_profiling(True)
    ex.execute([x])
    prof = ex.profile(False)
    ex.set_profiling(False)
    ms = sum(p[2] for p in prof)
    nbytes = 2 * x.numel() * 4
    d = plan.describe_steps(False).splitlines()[0]
    print(f"{expr:24s} {x.numel()*4/1e6:8.1f} MB  kernel {ms*1e3:8.1f} us  {nbytes/(ms*1e-3)/1e9:7.0f} GB/s"
          f"  (call {ms_call*1e3:7.1f} us)  {d}")
    del ex
