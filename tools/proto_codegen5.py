"""Prototype 5 of the per-matrix code generator: the full kernel shape.

CTA = W consumer warps + 1 TMA producer warp.  CTA tile = 64·W columns of N (each lane 2 columns).
The producer streams X[k0:k0+KC, tile] as W/4 TMA boxes of {256 cols × KC rows} per chunk into an
S-stage mbarrier ring.  Consumers run the panel's generated straight-line code: per union column one
LDS.64 of the lane's X pair (immediate offset; LDS issued PF columns ahead) and one FFMA2 with the
weight as a broadcast immediate per nonzero, accumulators a<r> named statically per row.

usage: python tools/proto_codegen5.py R K W KC S PF out.ptx [density]
"""
import random
import struct
import sys

R, K, W, KC, S, PF = (int(a) for a in sys.argv[1:7])
out = sys.argv[7]
dens = float(sys.argv[8]) if len(sys.argv) > 8 else 0.1
rng = random.Random(0)
NB = W                    # TMA boxes per chunk (64 columns each, one per consumer warp)
BOX = KC * 256            # bytes per box
STAGE = NB * BOX
NCH = (K + KC - 1) // KC
BAR = S * STAGE           # barrier area offset


def imm2(v):
    u = struct.unpack("<I", struct.pack("<f", v))[0]
    return "0x%08X%08X" % (u, u)


cols = []
for c in range(K):
    rows = [r for r in range(R) if rng.random() < dens]
    if rows:
        cols.append((c, rows))
nnz = sum(len(r) for _, r in cols)
T = (W + 1) * 32

L = [".version 8.8", ".target sm_100a", ".address_size 64", ""]
L.append(".extern .shared .align 1024 .b8 smem[];")
L.append(".visible .entry cg(.param .align 64 .b8 tmap[128], .param .u64 pY, .param .u32 ldy4, .param .u32 N)")
L.append(f".maxntid {T}, 1, 1")
L.append(".minnctapersm 1")
L.append("{")
L.append(f"  .reg .b64 a<{R}>; .reg .b64 x<{PF + 1}>; .reg .b64 ww, py, pc, t64, tm; .reg .b32 r<32>; .reg .pred p<8>;")
L.append("  mov.u32 r0, %tid.x; shr.u32 r1, r0, 5; and.b32 r2, r0, 31;")  # r1 warp, r2 lane
L.append(f"  mov.u32 r3, %ctaid.x; mul.lo.u32 r4, r3, {64 * W};")  # n0
L.append("  mov.u32 r5, smem;")  # smem base
L.append("  setp.ne.u32 p0, r0, 0; @p0 bra INITDONE;")
for s in range(S):
    L.append(f"  mbarrier.init.shared::cta.b64 [r5+{BAR + 8 * s}], 1;")
    L.append(f"  mbarrier.init.shared::cta.b64 [r5+{BAR + 8 * (S + s)}], {W};")
L.append("  fence.mbarrier_init.release.cluster;")
L.append("INITDONE:")
L.append("  bar.sync 0;")
L.append(f"  setp.ne.u32 p1, r1, {W}; @p1 bra CONSUMER;")
# ---------------- producer
L.append("  setp.ne.u32 p2, r2, 0; @p2 bra DONE;")
L.append("  mov.b64 tm, tmap; cvta.param.u64 tm, tm;")
for j in range(NCH):
    s = j % S
    if j >= S:
        par = ((j // S) - 1) & 1
        L.append(f"WE{j}: mbarrier.try_wait.parity.shared::cta.b64 p3, [r5+{BAR + 8 * (S + s)}], {par}; @!p3 bra WE{j};")
    L.append(f"  mbarrier.arrive.expect_tx.shared::cta.b64 _, [r5+{BAR + 8 * s}], {STAGE};")
    for b in range(NB):
        L.append(f"  add.u32 r6, r4, {64 * b}; add.u32 r7, r5, {s * STAGE + b * BOX}; add.u32 r8, r5, {BAR + 8 * s};")
        L.append(f"  cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [r7], [tm, {{r6, {j * KC}}}], [r8];")
L.append("  bra DONE;")
# ---------------- consumer
L.append("CONSUMER:")
# lane base: box = warp/4, col within box = (warp%4)*64 + 2*lane  -> byte offset
L.append("  shl.b32 r11, r2, 1;")
L.append(f"  mul.lo.u32 r9, r1, {BOX}; shl.b32 r10, r2, 3; add.u32 r9, r9, r10; add.u32 r12, r5, r9;")  # r12 = x base
for i in range(R):
    L.append(f"  mov.b64 a{i}, 0;")
ci = 0
by_chunk = {}
for c, rows in cols:
    by_chunk.setdefault(c // KC, []).append((c, rows))
k = 0
for j in range(NCH):
    s = j % S
    par = (j // S) & 1
    L.append(f"WF{j}: mbarrier.try_wait.parity.shared::cta.b64 p4, [r5+{BAR + 8 * s}], {par}; @!p4 bra WF{j};")
    ch = by_chunk.get(j, [])
    offs = [s * STAGE + (c % KC) * 256 for c, _ in ch]
    for i in range(min(PF, len(ch))):
        L.append(f"  ld.shared.b64 x{i % (PF + 1)}, [r12+{offs[i]}];")
    for i, (c, rows) in enumerate(ch):
        if i + PF < len(ch):
            L.append(f"  ld.shared.b64 x{(i + PF) % (PF + 1)}, [r12+{offs[i + PF]}];")
        xr = f"x{i % (PF + 1)}"
        for r in rows:
            L.append(f"  mov.b64 ww, {imm2(rng.gauss(0, 0.05))}; fma.rn.f32x2 a{r}, ww, {xr}, a{r};")
    L.append("  bar.warp.sync -1;")
    L.append(f"  @!p5 bra NA{j};")
    L.append(f"  mbarrier.arrive.shared::cta.b64 _, [r5+{BAR + 8 * (S + s)}];")
    L.append(f"NA{j}:")
# predicate p5 (lane 0) must be set before the loop: insert after consumer setup
L.insert(L.index("CONSUMER:") + 1, "  setp.eq.u32 p5, r2, 0;")
# epilogue: store rows r to Y[r][n], n = n0 + warp*64 + 2*lane
L.append("  ld.param.u64 py, [pY]; ld.param.u32 r13, [ldy4]; ld.param.u32 r14, [N];")
L.append("  shl.b32 r15, r1, 6; add.u32 r15, r15, r4; add.u32 r15, r15, r11;")
L.append("  setp.ge.u32 p6, r15, r14; @p6 bra DONE;")
L.append("  mul.wide.u32 t64, r15, 4; add.u64 py, py, t64;")
for r in range(R):
    L.append(f"  mad.wide.u32 pc, r13, {r}, py; st.global.b64 [pc], a{r};")
L.append("DONE: ret;")
L.append("}")
open(out, "w").write("\n".join(L) + "\n")
print("nnz", nnz, "cols", len(cols), "smem", S * STAGE + 16 * S)
