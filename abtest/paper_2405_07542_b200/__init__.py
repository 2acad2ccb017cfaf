"""B200-native EMS-SD unpadded multi-sample verify step (arXiv 2405.07542).

The compute lives in lib/libspecdec_b200.so (CUDA, sm_100a) behind the C ABI
in include/specdec_b200.h; `specdec` is the Python mirror of the reference
`specdec` C++ API over that ABI.
"""
