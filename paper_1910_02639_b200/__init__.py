"""B200-native b-tree exact close-neighbor search (arXiv 1910.02639).

The compute path is the CUDA library ``libbtree.so`` (C ABI in
``include/btree.h``); ``btree`` is its thin ctypes binding.  ``datagen`` draws
the seeded synthetic inputs.  Nothing here imports ``oracle/``.
"""
from .btree import BtreeError, Tree, build, lib, profile, profile_enable, profile_reset, release_cache, search_host, set_exact_only  # noqa: F401
