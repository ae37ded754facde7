"""paper_2104_14186_b200 — B200-native (sm_100a) QDWHpartial-EIG / QDWHpartial-SVD.

The product is libqdwhg.so (paper_2104_14186_b200/csrc, C ABI in include/qdwhg.h);
``qdwh`` mirrors the reference's qdwh:: C++ API on top of it.
"""
__version__ = "0.1.0"
