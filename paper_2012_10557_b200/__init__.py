"""paper_2012_10557_b200 -- B200-native hot path of Ekya's thief scheduler (arXiv 2012.10557).

The product is ``libekya.so`` (C ABI: ``include/ekya.h``; sm_100a kernels in
``csrc/``).  ``ekya`` is its ctypes binding.  This package never imports the
CPU oracle (``oracle/``), and has no CPU compute path.
"""
from . import ekya  # noqa: F401

__all__ = ["ekya"]
