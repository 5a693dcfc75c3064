"""Seeded random parity sweep (GPU): random engines, exponents, kernel choices, request lengths,
host / device outputs, host chunk sizes, output kinds, skips and state save/restore -- every
word compared with the CPU oracle. Complements the targeted parity tests with combinations
nobody wrote down."""
import os
import random

import numpy as np
import pytest
import torch

import oracle_py
from paper_1501_07701_b200 import mtgp, tables

pytestmark = pytest.mark.gpu


def _mtgp_ref(sets, seeds, start, n):
    return oracle_py.mtgp_bulk(sets, seeds, n, skip=start, threads=len(sets))[0]


def _mt_ref(seeds, start, n):
    out = []
    for sd in seeds:
        o = oracle_py.MtOracle(None, sd)
        if start:
            o.fill(start)
        out.append(o.fill(n))
    return np.stack(out)


def _conv(u, kind):
    if kind == mtgp.U32:
        return u
    f = ((u >> 9) | 0x3F800000).astype(np.uint32)
    if kind == mtgp.F32_01OC:
        f = (np.float32(2.0) - f.view(np.float32)).view(np.uint32)
    return f


# MTGP_RANDOM_CASES widens the sweep for a one-off long run (profiles/r2/random_sweep_long.txt)
@pytest.mark.parametrize("case", range(int(os.environ.get("MTGP_RANDOM_CASES", "40"))))
def test_random_request_sequences(case, curand_sets):
    rnd = random.Random(1501 + case)
    engine = rnd.choice(["mtgp11213", "mtgp23209", "mtgp44497", "mt"])
    S = rnd.choice([1, 3, 7, 16])
    seeds = [rnd.getrandbits(32) for _ in range(S)]
    if engine == "mt":
        ctx = mtgp.MtContext([mtgp.mt19937_status()] * S, seeds)
        kernels = [0, 1]
    else:
        mexp = int(engine[4:])
        sets = rnd.sample(curand_sets, S) if mexp == 11213 else tables.synthetic_sets(mexp, S, first=rnd.randint(0, 50))
        ctx = mtgp.MtgpContext(sets, seeds)
        kernels = [0, 1, 2] + ([3] if mexp == 11213 else []) + [4]
    pos = 0
    saved = None
    with ctx:
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, rnd.choice([1 << 10, 1 << 14, 1 << 21]))
        # speculative next-call jumps on in two thirds of the cases (own generator: the cases'
        # request sequences stay what they were)
        ctx.set_option(mtgp.OPT_PREJUMP, random.Random(9000 + case).choice([0, 2, 2]))
        for _ in range(6):
            op = rnd.choice(["host", "host", "device", "skip", "save", "restore"])
            kern = rnd.choice(kernels)
            ctx.set_option(mtgp.OPT_KERNEL, kern)
            if op in ("host", "device"):
                kind = rnd.choice([mtgp.U32, mtgp.U32, mtgp.F32_12, mtgp.F32_01OC])
                if kern == 4 and kind != mtgp.U32:
                    kind = mtgp.U32  # v4 is u32-only (the planner falls back for floats otherwise)
                L = rnd.choice([1, 3, 4, 255, 256, 1000, 4096, 65536 + 4 * rnd.randint(0, 999), 300001])
                if kern in (3, 4):
                    L = max(4, L - L % 4)  # the register kernels need L % 4 == 0
                if op == "host":
                    ctx.set_option(mtgp.OPT_HOST_CHUNK, rnd.choice([1, 777, 4096, 1 << 18]))
                    got = ctx.generate_host(kind, L)
                else:
                    buf = torch.empty((S, L), dtype=torch.int32, device="cuda")
                    ctx.generate_device(kind, buf.data_ptr(), L)
                    ctx.sync()
                    got = buf.cpu().numpy().view(np.uint32)
                ref = _mt_ref(seeds, pos, L) if engine == "mt" else _mtgp_ref(sets, seeds, pos, L)
                assert np.array_equal(got, _conv(ref, kind)), (case, op, kern, kind, L, pos)
                pos += L
            elif op == "skip":
                k = rnd.choice([1, 100, 5000, 123457])
                ctx.skip(k)
                pos += k
            elif op == "save":
                saved = ctx.state_save() + (pos,)
            elif op == "restore" and saved is not None:
                ctx.state_restore(saved[0], saved[1])
                pos = saved[2]
