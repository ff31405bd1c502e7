"""Generates the 2^(k/128) table of csrc/glibc_exp.cuh (the table of glibc's `exp`): for k in
[0, 128), H = 2^(k/128) rounded to the nearest double and T = (2^(k/128) - H) / H rounded to the
nearest double, both from 80-digit decimal arithmetic; tab[2k] = bits(T), tab[2k+1] = bits(H) -
(k << 45). With --check LIBM, also reports whether the same 2 KB appear in that libm."""
import struct
import sys
from decimal import Decimal, getcontext


def table():
    getcontext().prec = 80
    ln2 = Decimal(2).ln()
    out = []
    for k in range(128):
        v = (Decimal(k) / 128 * ln2).exp()
        h = float(v)  # float(Decimal) rounds to nearest
        t = float((v - Decimal(h)) / Decimal(h))
        out.append(struct.unpack("<Q", struct.pack("<d", t))[0])
        out.append((struct.unpack("<Q", struct.pack("<d", h))[0] - (k << 45)) & (2**64 - 1))
    return out


if __name__ == "__main__":
    tab = table()
    if len(sys.argv) > 2 and sys.argv[1] == "--check":
        blob = open(sys.argv[2], "rb").read()
        print("found in", sys.argv[2], ":", struct.pack("<256Q", *tab) in blob)
    else:
        for i in range(0, 256, 4):
            print("    " + ", ".join("0x%016xull" % t for t in tab[i:i + 4]) + ",")
