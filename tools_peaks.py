import ctypes, sys
sys.path.insert(0, '.')
from paper_1811_00778_b200 import _lib
L = _lib.lib()
names = {0: "IMAD", 1: "IMAD.HI", 2: "IMAD.WIDE(+add)", 3: "IADD+UMIN", 4: "csub-mask", 5: "IADD3", 6: "DFMA", 7: "IMAD.WIDE||DFMA (both counted)",
         8: "Harvey butterfly, 16 warps/SMSP", 9: "Harvey butterfly, 4 warps/SMSP"}
for k in range(10):
    v = ctypes.c_double()
    _lib.check(L.hcnn_int_peak(0, k, ctypes.byref(v)))
    print(f"{k} {names[k]:32s} {v.value/1e12:7.2f} T/s")
