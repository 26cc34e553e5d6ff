"""B200 (sm_100a) packed approximate overlap-save convolution (arXiv 1201.3018).

The product is ``libpackedconv.so`` (C ABI in include/packedconv.h); ``binding`` is its
thin ctypes binding and ``workloads`` the seeded synthetic inputs.  Importing the package
does not load the library; ``binding.load()`` does, and raises if it is not built.
"""
__all__ = ["binding", "workloads", "build"]
