"""B200-native (sm_100a) PD+IPC iteration of arXiv 2312.02999 behind a C ABI.

The product is libpd_ipc.so (csrc/, include/pd_ipc.h); `pd_ipc` is its thin ctypes binding.
"""
