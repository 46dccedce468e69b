"""B200-native EGT (dilated entropy) + CFR solver for poker endgames (arXiv:1810.03063).

The hot path lives in the CUDA library ``lib/libegt_b200.so`` (sources in
``csrc/``, C ABI in ``include/egt_b200.h``); ``binding`` is a thin ctypes layer
over it.  ``workloads`` holds the seeded synthetic inputs.  Importing this
package does not load the library; the first solver call does, and fails loudly
if it is missing.
"""
from .binding import (CFR_PLUS, CFR_RM, CFR_RMP, EGT_AS, EGT_BALANCED, EGT_THEORY, KUHN, LEDUC,  # noqa: F401
                      RIVER, EGTError, Game, load_game, load_library, pool_trim)
from .solve import solve  # noqa: F401
