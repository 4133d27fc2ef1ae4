"""B200-native (sm_100a) hot path of arXiv 2211.09938's saliency-gated
progressive hologram synthesis (reference: wavecgh 0.1.0).

Layers: csrc/ (CUDA kernels + the C ABI, include/wcgh.h) -> _lib (ctypes)
-> stages / hologram / tiles (host mirror of the reference interface).
"""
__version__ = "0.1.0"
