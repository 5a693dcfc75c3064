"""cuRAND's own device MTGP32 as a second, on-device independent pin.

oracle/_ref/curand_device (oracle/curand_device.cu; test infrastructure) runs cuRAND's
device-API curand() kernel -- one curandStateMtgp32_t per 256-thread block, its 1024-word ring
(curand_mtgp32_kernel.h:196-228) -- over the 200 certified MTGP32-11213 sets with cuRAND's own
state setup (curandMakeMTGP32Constants / curandMakeMTGP32KernelState: stream i seeded with
(u32)(seed ^ seed >> 32) + i + 1). The product path (C-ABI, default auto plan: gen3 warp teams
with jump-ahead pieces) given the same sets and seeds must produce the same words.
"""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1501_07701_b200 import mtgp, tables

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "curand_device"
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not BIN.exists(), reason="make -C oracle device")]


def _curand(L: int, seed: int) -> dict:
    r = subprocess.run([str(BIN), "words", str(L), str(seed)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout)


@pytest.mark.parametrize("seed", [0, 0x1234_5678_9ABC])
def test_all_200_sets_equal_curand_device(seed):
    L = 1 << 20
    ref = _curand(L, seed)
    sets = tables.load_curand_11213()
    seeds = [st["seed"] for st in ref["streams"]]
    assert seeds[:2] == [((seed ^ (seed >> 32)) + 1) & 0xFFFFFFFF, ((seed ^ (seed >> 32)) + 2) & 0xFFFFFFFF]
    with mtgp.MtgpContext(sets, seeds) as ctx:
        ctx.set_option(mtgp.OPT_CHECKSUM, 1)
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 16)  # split every stream: jump-ahead pieces too
        w = ctx.fill_u32(L)
        cks = ctx.checksums()
        assert ctx.last_plan()[0] > 200
    for s, st in enumerate(ref["streams"]):
        assert list(w[s, :8]) == st["first"], s
        assert int(w[s, -1]) == st["last"], s
        assert int(w[s].astype(np.uint64).sum()) == st["sum64"], s
        assert int(np.bitwise_xor.reduce(w[s])) == st["xor32"], s
        assert (cks[s][0], cks[s][1], cks[s][2]) == (st["sum64"], st["xor32"], L), s
