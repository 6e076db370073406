"""libraas — B200-native page-based RaaS decode (arXiv 2502.11147).

The compute path is ``libraas.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/raas.h``); ``paper_2502_11147_b200.raas`` is the thin ctypes binding with the
same names.  Importing this package does not load the library; ``raas.lib()`` does, and
fails loudly if it is missing.
"""

__all__ = ["raas", "synth"]
