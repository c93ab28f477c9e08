"""paper_2402_18789_b200 -- B200-native co-serving iteration (FlexLLM, arXiv 2402.18789).

The product is libcoserve_cuda.so (sm_100a kernels + C++ engine behind the C ABI in
include/coserve_cuda.h).  This Python package is the thin host mirror used by tests and
bench.py: a ctypes binding (_lib), an in-tree build (build) and the engine wrapper.
"""
__all__ = ["build", "_lib"]
