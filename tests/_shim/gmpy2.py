"""Test-only stand-in for gmpy2 when importing the reference (hefir) here.

The reference uses gmpy2 only as `gmpy2.mpz(x)` around one exact big-integer
multiply (ring.py:324-326); Python ints give the same exact integers, slower.
"""
mpz = int
