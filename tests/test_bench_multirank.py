"""The driver's multi-GPU bench command line (`python bench.py --gpus N` without torchrun
variables: bench.py re-launches itself under torch.distributed.run) exercised end to end on
ONE GPU: CE_BENCH_SHARE_GPU=1 puts both ranks on device 0 with gloo collectives (NCCL refuses
two ranks per device); batch sharding, the factor-gradient all-reduce and the max-over-ranks
timing all run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_gpus2_self_launch_on_one_gpu():
    env = dict(os.environ, CE_BENCH_SHARE_GPU="1")
    env.pop("RANK", None)
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cfg3",
                        "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == "weak"
