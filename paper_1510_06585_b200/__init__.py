"""B200-native Marrow hot path (arxiv 1510.06585): skeleton computation trees
over partitioned inputs, executed by hand-written sm_100a kernels in
libmarrow.so (C-ABI: include/marrow.h).  ``marrow`` is the thin ctypes
binding; ``trees`` builds the paper's benchmark trees from built-in kernels."""
from . import marrow  # noqa: F401
from . import trees  # noqa: F401

marrow.lib()  # fail loudly at import if the native library is missing
