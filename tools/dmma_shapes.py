"""FP64 MMA shapes on this GPU: throughput (all SMs, independent accumulators)
and dependent-chain latency (one warp) of m8n8k4 / m16n8k8 / m16n8k16."""
import ctypes
import os
lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "libfp64probe.so"))
lib.probe_dmma_peak.restype = ctypes.c_double
lib.probe_dmma_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
lib.probe_dmma_latency.restype = ctypes.c_double
lib.probe_dmma_latency.argtypes = [ctypes.c_int, ctypes.c_int]
ms = ctypes.c_float()
for which, name in ((0, "m8n8k4"), (2, "m16n8k8"), (1, "m16n8k16")):
    tf = lib.probe_dmma_peak(which, 4000 if which else 16000, ctypes.byref(ms))
    lat = lib.probe_dmma_latency(which, 4096)
    print(f"{name:9s} {tf:6.2f} TFLOP/s ({ms.value:.2f} ms)   dependent chain {lat:6.1f} cycles/MMA")
