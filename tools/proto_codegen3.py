"""Prototype 3 of the per-matrix code generator: V = 2 columns per lane, FFMA2 with the weight as a
broadcast immediate (ptxas folds a 64-bit constant with equal halves into `FFMA2 R, R.F32x2, imm, R`),
accumulators named statically per row, X pairs prefetched D columns ahead through a running 64-bit
pointer, basic blocks split every B columns by a never-taken uniform branch (bounds ptxas time).

usage: python tools/proto_codegen3.py R K D B out.ptx [threads]
"""
import random
import struct
import sys

R, K, D, B = (int(a) for a in sys.argv[1:5])
out = sys.argv[5]
THREADS = int(sys.argv[6]) if len(sys.argv) > 6 else 384
rng = random.Random(0)


def imm2(v):
    u = struct.unpack("<I", struct.pack("<f", v))[0]
    return "0x%08X%08X" % (u, u)


cols = []
for c in range(K):
    rows = [r for r in range(R) if rng.random() < 0.1]
    if rows:
        cols.append((c, rows))
nnz = sum(len(r) for _, r in cols)

L = [".version 8.8", ".target sm_100a", ".address_size 64", ""]
L.append(".visible .entry cg(.param .u64 pX, .param .u64 pY, .param .u32 ldx4, .param .u32 ldy4, .param .u32 N, .param .u32 never)")
L.append(f".maxntid {THREADS}, 1, 1")
L.append(".minnctapersm 1")
L.append("{")
L.append(f"  .reg .b64 a<{R}>; .reg .b64 x<{D}>; .reg .b64 ww, px, py, pc, pl, stride, t64; .reg .b32 r<16>; .reg .pred p<4>, pn;")
L.append("  ld.param.u64 px, [pX]; ld.param.u64 py, [pY]; ld.param.u32 r0, [ldx4]; ld.param.u32 r1, [ldy4];")
L.append("  ld.param.u32 r2, [N]; ld.param.u32 r3, [never]; setp.ne.u32 pn, r3, 0;")
L.append(f"  mov.u32 r4, %ctaid.x; mov.u32 r7, %tid.x; mad.lo.u32 r8, r4, {THREADS}, r7; shl.b32 r8, r8, 1;")
L.append("  sub.u32 r9, r2, 2; min.u32 r10, r8, r9;")
L.append("  mul.wide.u32 t64, r10, 4; add.u64 px, px, t64; cvt.u64.u32 stride, r0;")
for i in range(R):
    L.append(f"  mov.b64 a{i}, 0;")
# pl = load pointer (column of the next load); loads walk the union columns in order
L.append(f"  mad.wide.u32 pl, r0, {cols[0][0]}, px;")
prev = cols[0][0]


def emit_load(i, reg):
    global prev
    c = cols[i][0]
    d = c - prev
    if d == 1:
        L.append("  add.s64 pl, pl, stride;")
    elif d > 1:
        L.append(f"  mad.wide.u32 pl, r0, {d}, pl;")
    prev = c
    L.append(f"  ld.global.nc.L1::no_allocate.b64 {reg}, [pl];")


for i in range(min(D, len(cols))):
    emit_load(i, f"x{i}")
for i, (c, rows) in enumerate(cols):
    xr = f"x{i % D}"
    for r in rows:
        L.append(f"  mov.b64 ww, {imm2(rng.gauss(0, 0.05))}; fma.rn.f32x2 a{r}, ww, {xr}, a{r};")
    if i + D < len(cols):
        emit_load(i + D, xr)
    if B and (i + 1) % B == 0:
        L.append(f"  @pn bra DONE;")
L.append("  setp.ge.u32 p1, r8, r2; @p1 bra DONE;")
L.append("  mul.wide.u32 t64, r8, 4; add.u64 py, py, t64;")
for r in range(R):
    L.append(f"  mad.wide.u32 pc, r1, {r}, py; st.global.b64 [pc], a{r};")
L.append("DONE: ret;")
L.append("}")
open(out, "w").write("\n".join(L) + "\n")
print("nnz", nnz, "cols", len(cols))
