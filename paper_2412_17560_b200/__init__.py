"""GQSA (arXiv 2412.17560) decode hot path, B200-native (sm_100a).

The product is the C-ABI library ``lib/libgqsa.so`` (include/gqsa.h); this
package holds its thin ctypes binding (:mod:`.gqsa`) and the seeded synthetic
input generators (:mod:`.synth`).
"""
