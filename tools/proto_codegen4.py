"""Prototype 4: module with P panel .funcs + one entry switching on the panel (compile-time probe for
ptxas --split-compile).  Consumer body as in proto 3 but reading X pairs from shared memory with
immediate offsets (the TMA-staged tile), weights as FFMA2 broadcast immediates.

usage: python tools/proto_codegen4.py R K P out.ptx
"""
import random
import struct
import sys

R, K, P = (int(a) for a in sys.argv[1:4])
out = sys.argv[4]
rng = random.Random(0)
ROWB = 3072  # bytes per staged X row (768 columns)
KC = 16
S = 4


def imm2(v):
    u = struct.unpack("<I", struct.pack("<f", v))[0]
    return "0x%08X%08X" % (u, u)


L = [".version 8.8", ".target sm_100a", ".address_size 64", ""]
for p in range(P):
    L.append(f".func panel{p}(.param .u32 xs)")
    L.append("{")
    L.append(f"  .reg .b64 a<{R}>; .reg .b64 x<4>; .reg .b32 xb; .reg .b64 ww;")
    L.append("  ld.param.u32 xb, [xs];")
    for i in range(R):
        L.append(f"  mov.b64 a{i}, 0;")
    cols = []
    for c in range(K):
        rows = [r for r in range(R) if rng.random() < 0.1]
        if rows:
            cols.append((c, rows))
    for i, (c, rows) in enumerate(cols):
        j = c // KC
        off = (j % S) * KC * ROWB + (c % KC) * ROWB
        L.append(f"  ld.shared.b64 x{i % 4}, [xb+{off}];")
        for r in rows:
            L.append(f"  mov.b64 ww, {imm2(rng.gauss(0, 0.05))}; fma.rn.f32x2 a{r}, ww, x{i % 4}, a{r};")
    for r in range(R):
        L.append(f"  st.shared.b64 [xb+{8 * r}], a{r};")
    L.append("  ret;")
    L.append("}")
L.append(".visible .entry cg(.param .u32 pan)")
L.append(".maxntid 416, 1, 1")
L.append("{")
L.append("  .reg .b32 p, xs; .reg .pred q; .shared .align 16 .b8 buf[4096];")
L.append("  ld.param.u32 p, [pan]; mov.u32 xs, buf;")
L.append("  .param .u32 arg;")
L.append("  st.param.u32 [arg], xs;")
for p in range(P):
    L.append(f"  setp.eq.u32 q, p, {p}; @q call panel{p}, (arg);")
L.append("  ret;")
L.append("}")
open(out, "w").write("\n".join(L) + "\n")
