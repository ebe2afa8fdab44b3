"""Prototype 2 of the per-matrix code generator: V = 2 columns per lane, FFMA2 (fma.rn.f32x2) with
the weight broadcast from a uniform 16-byte load of the panel's weight stream (4 weights per load),
accumulator registers named statically per row.  One PTX .entry per panel.

usage: python tools/proto_codegen2.py R K D WAHEAD out.ptx
"""
import random
import struct
import sys

R, K, D, WA = (int(a) for a in sys.argv[1:5])
out = sys.argv[5]
rng = random.Random(0)
THREADS = 384

cols = []
for c in range(K):
    rows = [r for r in range(R) if rng.random() < 0.1]
    if rows:
        cols.append((c, rows))
nnz = sum(len(r) for _, r in cols)

L = [".version 8.8", ".target sm_100a", ".address_size 64", ""]
L.append(".visible .entry cg(.param .u64 pX, .param .u64 pY, .param .u64 pW, .param .u32 ldx4, .param .u32 ldy4, .param .u32 N)")
L.append(f".maxntid {THREADS}, 1, 1")
L.append(".minnctapersm 1")
L.append("{")
L.append(f"  .reg .b64 a<{R}>; .reg .b64 x<{D}>; .reg .f32 w<{4 * WA}>; .reg .b64 ww, px, py, pw, pc, t64; .reg .b32 r<16>; .reg .pred p<4>;")
L.append("  ld.param.u64 px, [pX]; ld.param.u64 py, [pY]; ld.param.u64 pw, [pW]; ld.param.u32 r0, [ldx4]; ld.param.u32 r1, [ldy4];")
L.append("  ld.param.u32 r2, [N];")
L.append(f"  mov.u32 r4, %ctaid.x; mov.u32 r7, %tid.x; mad.lo.u32 r8, r4, {THREADS}, r7; shl.b32 r8, r8, 1;")  # n (pair)
L.append("  sub.u32 r9, r2, 2; min.u32 r10, r8, r9;")
L.append("  mul.wide.u32 t64, r10, 4; add.u64 px, px, t64;")
for i in range(R):
    L.append(f"  mov.b64 a{i}, 0;")
# weight groups
ngroups = (nnz + 3) // 4


def wload(g):
    return f"  ld.global.nc.v4.f32 {{w{4 * (g % WA)}, w{4 * (g % WA) + 1}, w{4 * (g % WA) + 2}, w{4 * (g % WA) + 3}}}, [pw+{16 * g}];"


for g in range(min(WA, ngroups)):
    L.append(wload(g))
for i in range(min(D, len(cols))):
    L.append(f"  mad.wide.u32 pc, r0, {cols[i][0]}, px; ld.global.nc.L1::no_allocate.v2.f32 {{%tmpa, %tmpb}}, [pc];".replace("{%tmpa, %tmpb}", f"x{i}"))
k = 0
for i, (c, rows) in enumerate(cols):
    xr = f"x{i % D}"
    for r in rows:
        g, s = divmod(k, 4)
        L.append(f"  mov.b64 ww, {{w{4 * (g % WA) + s}, w{4 * (g % WA) + s}}}; fma.rn.f32x2 a{r}, ww, {xr}, a{r};")
        k += 1
        if s == 3 and g + WA < ngroups:
            L.append(wload(g + WA))
    if i + D < len(cols):
        L.append(f"  mad.wide.u32 pc, r0, {cols[i + D][0]}, px; ld.global.nc.L1::no_allocate.b64 {xr}, [pc];")
L.append("  setp.ge.u32 p1, r8, r2; @p1 bra DONE;")
L.append("  mul.wide.u32 t64, r8, 4; add.u64 py, py, t64;")
for r in range(R):
    L.append(f"  mad.wide.u32 pc, r1, {r}, py; st.global.b64 [pc], a{r};")
L.append("DONE: ret;")
L.append("}")
s = "\n".join(L) + "\n"
s = s.replace("ld.global.nc.L1::no_allocate.v2.f32 x", "ld.global.nc.L1::no_allocate.b64 x")
open(out, "w").write(s)
print("nnz", nnz, "cols", len(cols))
