"""Prototype of the per-matrix code generator — compile-time / SASS-quality probe.

Generates one PTX .entry for P panels of R rows of a synthetic 90 %-sparse matrix: per union column
one 64-bit address mad + one LDG of X (prefetched D columns ahead) and one FFMA per nonzero with the
weight as an immediate into the accumulator register of its row.

usage: python tools/proto_codegen.py R K P D out.ptx
"""
import random
import struct
import sys

R, K, P, D = (int(a) for a in sys.argv[1:5])
out = sys.argv[5]
SYNC = int(sys.argv[6]) if len(sys.argv) > 6 else 0
rng = random.Random(0)


def f2h(v):
    return "0f%08X" % struct.unpack("<I", struct.pack("<f", v))[0]


L = [".version 8.8", ".target sm_100a", ".address_size 64", ""]
L.append(".visible .entry cg(.param .u64 pX, .param .u64 pY, .param .u32 ldx4, .param .u32 ldy4, .param .u32 N, .param .u32 npan)")
L.append(".maxntid 384, 1, 1")
L.append(".minnctapersm 1")
L.append("{")
L.append(f"  .reg .f32 a<{R}>; .reg .f32 x<{D}>; .reg .b64 px, py, pc, t64; .reg .b32 r<16>; .reg .pred p<4>;")
L.append("  ld.param.u64 px, [pX]; ld.param.u64 py, [pY]; ld.param.u32 r0, [ldx4]; ld.param.u32 r1, [ldy4];")
L.append("  ld.param.u32 r2, [N]; ld.param.u32 r3, [npan];")
L.append("  mov.u32 r4, %ctaid.x; rem.u32 r5, r4, r3; div.u32 r6, r4, r3;")  # r5 = panel, r6 = tile
L.append("  mov.u32 r7, %tid.x; mad.lo.u32 r8, r6, 384, r7;")  # n
L.append("  sub.u32 r9, r2, 1; min.u32 r10, r8, r9;")  # clamped n
L.append("  mul.wide.u32 t64, r10, 4; add.u64 px, px, t64;")
for i in range(R):
    L.append(f"  mov.f32 a{i}, 0f00000000;")
nf = 0
for pan in range(P):
    L.append(f"  setp.ne.u32 p0, r5, {pan}; @p0 bra PAN{pan + 1};")
    cols = []
    for c in range(K):
        rows = [r for r in range(R) if rng.random() < 0.1]
        if rows:
            cols.append((c, rows))
    for i in range(min(D, len(cols))):
        L.append(f"  mad.wide.u32 pc, r0, {cols[i][0]}, px; ld.global.nc.L1::no_allocate.f32 x{i}, [pc];")
    for i, (c, rows) in enumerate(cols):
        xr = f"x{i % D}"
        for r in rows:
            L.append(f"  fma.rn.f32 a{r}, {xr}, {f2h(rng.gauss(0, 0.05))}, a{r};")
            nf += 1
        if i + D < len(cols):
            L.append(f"  mad.wide.u32 pc, r0, {cols[i + D][0]}, px; ld.global.nc.L1::no_allocate.f32 {xr}, [pc];")
        if SYNC and (i + 1) % SYNC == 0:
            L.append("  bar.sync 0;")
    L.append("  bra EPI;")
    L.append(f"PAN{pan + 1}:")
L.append("EPI:")
L.append("  setp.ge.u32 p1, r8, r2; @p1 bra DONE;")
L.append("  mul.wide.u32 t64, r8, 4; add.u64 py, py, t64;")
for r in range(R):
    L.append(f"  mad.wide.u32 pc, r1, {r}, py; st.global.f32 [pc], a{r};")
L.append("DONE: ret;")
L.append("}")
open(out, "w").write("\n".join(L) + "\n")
print("fma", nf, "lines", len(L))
