"""Random conv_einsum spec generator in the spirit of SPEC.md:563-565 (test helper)."""
import numpy as np

POOL = list("abcdefg")
MODES = ["full", "same", "valid", "circular"]


def random_spec(rng, n_min=2, n_max=5, dmax=6, max_atoms=4):
    n = int(rng.integers(n_min, n_max + 1))
    ins = []
    for _ in range(n):
        k = int(rng.integers(1, max_atoms + 1))
        ins.append(list(rng.choice(POOL, size=k, replace=False)))
    present = []
    for s in ins:
        for a in s:
            if a not in present:
                present.append(a)
    out = [a for a in present if rng.random() < 0.5]
    rng.shuffle(out)
    occ = {a: sum(a in s for s in ins) for a in present}
    convs = [a for a in out if occ[a] >= 2 and rng.random() < 0.5]
    mode = MODES[int(rng.integers(0, 4))]
    base = {a: int(rng.integers(1, dmax + 1)) for a in present}
    dims = []
    for s in ins:
        d = []
        for a in s:
            if a in convs and occ[a] == 2:
                d.append(int(rng.integers(1, dmax + 1)))
            else:
                d.append(base[a])
        dims.append(d)
    expr = ",".join("".join(s) for s in ins) + "->" + "".join(out) + ("|" + "".join(convs) if convs else "")
    return expr, dims, mode
