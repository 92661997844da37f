"""Integer / FP64 pipe probes (hcnn_int_peak kinds 0-15): the measured rates behind DESIGN.md section 4."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_00778_b200 import _lib
L = _lib.lib()
names = {0: "IMAD", 1: "IMAD.HI", 2: "IMAD.WIDE(+add)", 3: "IADD+UMIN", 4: "csub-mask", 5: "IADD3", 6: "DFMA", 7: "IMAD.WIDE||DFMA (both counted)",
         8: "Harvey butterfly, 16 warps/SMSP", 9: "Harvey butterfly, 4 warps/SMSP",
         10: "butterfly, fp64 quotient", 11: "Shoup multiplies only", 12: "butterfly adds only",
         13: "11-term dot mod p, IMAD.WIDE+REDC", 14: "11-term dot mod p, FP64 split", 15: "11-term dot, alternating"}
for k in range(16):
    v = ctypes.c_double()
    _lib.check(L.hcnn_int_peak(0, k, ctypes.byref(v)))
    print(f"{k} {names[k]:32s} {v.value/1e12:7.2f} T/s")
