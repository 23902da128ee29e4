"""B200-native SOFA exact k-NN path (arxiv 2411.17483).

The product is libsofa.so (include/sofa.h, kernels in csrc/); `sofa` is its ctypes binding,
`index.SofaIndex` the user API, `distributed` the one-process-per-GPU sharding, `datagen`
the seeded synthetic workloads.
"""
__all__ = ["datagen", "sofa", "index", "distributed", "build"]
