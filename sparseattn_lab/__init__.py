"""``sparseattn_lab`` drop-in shim: the reference package's hot-path module names
(``sparseattn_lab.masker``, ``.attention``, ``.numerics``; /root/reference/pkg/src/
sparseattn_lab) resolved to the B200 implementation in ``paper_2602_13515_b200``.

Reference callers switch by putting this directory's parent on ``sys.path`` (or installing
it) instead of the reference: ``from sparseattn_lab import masker as mk`` then returns the
GPU module itself (``mk is paper_2602_13515_b200.masker``), so names, argument meaning,
result types (numpy in -> read-only numpy out) and exceptions are the reference's
(SURVEY.md §8b).  Only the hot path is provided; the reference's flow-matching model,
analysis, CLI and SPT2 I/O are out of scope.
"""

import sys as _sys

from paper_2602_13515_b200 import attention, masker, numerics  # noqa: F401

__version__ = "0.1.0"

for _name, _mod in (("masker", masker), ("attention", attention), ("numerics", numerics)):
    _sys.modules[f"{__name__}.{_name}"] = _mod
