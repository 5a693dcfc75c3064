"""paper_1501_07701_b200 -- B200-native MTGP32 bulk generation (arXiv 1501.07701's GPU generator).

Layout:
  csrc/            CUDA sm_100a kernels + the C-ABI (include/mtgp_b200.h) -> libmtgp_b200.so:
                   generation (v3 register ring for 11213, v4 templated on N for 23209/44497,
                   v2 shared-memory ring, v1 CTA-per-set, Engine::mt), jump-ahead planner,
                   device-side stat tests, certification
  tables.py        parameter-set tables (cuRAND 11213 import, synthetic sets, status files)
  mtgp.py          thin ctypes binding of the C-ABI (MtgpContext, MtContext) for tests / bench.py
  stattests.py     the reference's stat tests + campaign grid over the C-ABI (GPU)
  shard.py         multi-GPU set partitioning and the checksum gather

The C++ drop-in for the reference's generation path (GpuWordSource : WordSource,
make_word_source for Engine::mtgp32) lives in include/twistsieve_b200/ and is built into
libtwistsieve_b200.so on top of the same C-ABI.
"""
from . import tables  # noqa: F401

__all__ = ["tables"]
