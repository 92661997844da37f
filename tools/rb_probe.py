"""Which ring degrees take the relinearisation over R by default: for N =
2^13, 2^14, 2^15 with 6 primes, print N, the default NTT variant, the digit
count and hcnn_ctx_query(HCNN_Q_RELIN_RBASIS).

    python tools/rb_probe.py
"""
import numpy as np, sys
sys.path.insert(0,'.')
from paper_1811_00778_b200 import bfv as B, engine as E, _lib
for n in (8192, 16384, 32768):
    P=[]; c=(1<<30)//(2*n)
    while len(P)<6:
        p=c*2*n+1
        if all(p%d for d in range(3,int(p**.5)+1,2)): P.append(p)
        c-=1
    params=B.BfvParams(B.RnsContext(n,P),65537)
    g=E.context_for(params)
    print(n, g.variant(), g.D, _lib.lib().hcnn_ctx_query(g.handle,8))
