"""paper_2207_09442_b200 -- B200-native batched pose-graph GN/LM with implicit backward.

The hot path of Theseus (arXiv 2207.09442) behind the C ABI of include/dnls.h, implemented
in hand-written CUDA for sm_100a (csrc/).  Python here is argument marshalling
(``dnls``), the autograd layer (``layer``) and batch sharding over torch.distributed
(``parallel``).  There is no CPU compute path.
"""
from . import dnls  # noqa: F401
from ._lib import LIB_PATH, header_symbols, lib  # noqa: F401
