"""Dense vs 2:4-sparse tcgen05 int8 MMA throughput on all SMs (sparse_mma_rate.cu)."""
import ctypes
import json
import os

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "sparse_mma_rate.so"))
out = {}
for sparse in (0, 1):
    ms, cyc = ctypes.c_float(0), ctypes.c_double(0)
    iters = 20000
    rc = lib.run(sparse, iters, 148, ctypes.byref(ms), ctypes.byref(cyc))
    k_logical = 64 if sparse else 32
    macs = 148 * 4 * iters * 128 * 256 * k_logical
    out["sparse" if sparse else "dense"] = {"rc": rc, "ms": ms.value, "cycles_per_mma": cyc.value,
                                            "logical_tops": 2 * macs / (ms.value / 1e3) / 1e12}
print(json.dumps(out))
