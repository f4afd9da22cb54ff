"""Physical constants.

eta0 = mu0 * c with mu0 = 4*pi*1e-7 (pre-2019 SI) and c = 299792458 m/s.
One fixed value on both sides of the parity check: the 2019-SI eta0 differs
by 1.3e-10 relative, which alone would exceed the 1e-10 matvec tolerance.
"""
import math

C0 = 299792458.0
MU0 = 4.0e-7 * math.pi
ETA0 = MU0 * C0          # 376.730313461771... ohm
