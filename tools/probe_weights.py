"""Runs the FP64 probe kernels (tools/fp64probe.cu).  Plain run: prints the
DFMA peak.  Under `ncu --metrics sm__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum`
the k_unary launches give the FP64 op weight of one exp / log / div call:
    w = (2*dfma + dadd + dmul) / (threads * reps) - loop overhead (1 dadd acc
    + 1 dadd arg) per call; parsed by tools/weights_from_ncu.py."""
import ctypes
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libfp64probe.so"))
lib.probe_dfma_peak.restype = ctypes.c_double
lib.probe_dfma_peak.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
THREADS, REPS = 128 * 148, 64
for which in (0, 1, 2):
    rc = lib.probe_unary(which, THREADS, REPS)
    assert rc == 0, rc
ms = ctypes.c_float()
for it in (2000, 20000, 50000):
    t = lib.probe_dfma_peak(it, ctypes.byref(ms))
    print(f"dfma peak iters={it}: {t:.2f} TFLOP/s in {ms.value:.2f} ms")
lib.probe_dmma_peak.restype = ctypes.c_double
lib.probe_dmma_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
for which, name in ((0, "m8n8k4"), (1, "m16n8k16")):
    t = lib.probe_dmma_peak(which, 4000, ctypes.byref(ms))
    print(f"dmma {name}: {t:.2f} TFLOP/s in {ms.value:.2f} ms")
print(f"THREADS={THREADS} REPS={REPS}")
sys.exit(0)
