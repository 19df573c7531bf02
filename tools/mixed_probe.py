"""Do the FP64 tensor pipe (DMMA) and the FP64 FMA pipe add up?"""
import ctypes
import os
lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "libfp64probe.so"))
lib.probe_mixed.restype = ctypes.c_double
lib.probe_mixed.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
lib.probe_dfma_peak.restype = ctypes.c_double
lib.probe_dfma_peak.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
ms = ctypes.c_float()
print("dfma only", lib.probe_dfma_peak(20000, ctypes.byref(ms)))
for nm, nf in ((4, 0), (0, 8), (4, 2), (4, 4), (4, 8), (2, 4), (1, 4), (4, 16)):
    t = lib.probe_mixed(4000, nm, nf, ctypes.byref(ms))
    print(f"mma {nm} dfma8x{nf}: {t:.2f} TFLOP/s ({ms.value:.2f} ms)")
