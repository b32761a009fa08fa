"""B200-native HogBatch skip-gram negative-sampling SGD step (arXiv 1611.06172).

The product is the C-ABI library `libw2v.so` (include/w2v.h); `binding` is its ctypes wrapper.
"""
