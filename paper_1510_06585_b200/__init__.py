"""B200-native Marrow hot path (arxiv 1510.06585): skeleton trees over
partitioned inputs, executed by hand-written sm_100a kernels (libmarrow.so)."""
