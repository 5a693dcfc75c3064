"""paper_1501_07701_b200 -- B200-native MTGP32 bulk generation (arXiv 1501.07701's GPU generator).

Layout:
  csrc/            CUDA sm_100a kernels + the C-ABI (include/mtgp_b200.h) -> libmtgp_b200.so
  tables.py        parameter-set tables (cuRAND 11213 import, synthetic sets, status files)
  mtgp.py          thin ctypes binding of the C-ABI (MtgpContext) used by tests and bench.py

The C++ drop-in for the reference's generation path (GpuWordSource : WordSource,
make_word_source for Engine::mtgp32) lives in include/twistsieve_b200/ and is built into
libtwistsieve_b200.so on top of the same C-ABI.
"""
from . import tables  # noqa: F401

__all__ = ["tables"]
