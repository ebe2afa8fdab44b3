"""Prototype 6 of the per-matrix code generator: proto5 with per-warp K rotation.

Measured on proto5 (gpurun_out/cg5*.log, ncu): straight-line generated code is instruction-fetch
bound ("no_instruction" = 12 of 17.5 cycles per issued instruction) when all warps of the SM execute
the same code in lockstep (one fetch stream per SM).  Here consumer warp w starts at K chunk
w·NCH/W and wraps around, so the W warps sit at W different places of the code: W independent fetch
streams.  The stage ring is indexed by the logical step (same for all warps); the producer loads, for
step j, box w with chunk (j + off_w) mod NCH.

usage: python tools/proto_codegen6.py R K W KC S PF out.ptx [density] [rotate=1]
"""
import random
import struct
import sys

R, K, W, KC, S, PF = (int(a) for a in sys.argv[1:7])
out = sys.argv[7]
dens = float(sys.argv[8]) if len(sys.argv) > 8 else 0.1
rotate = int(sys.argv[9]) if len(sys.argv) > 9 else 1
assert S & (S - 1) == 0
LS = S.bit_length() - 1
rng = random.Random(0)
BOX = KC * 256            # bytes per box (KC rows x 64 columns fp32)
STAGE = W * BOX
NCH = (K + KC - 1) // KC
BAR = S * STAGE


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
offs = [(w * NCH // W) if rotate else 0 for w in range(W)]

L = [".version 8.8", ".target sm_100a", ".address_size 64", ""]
L.append(".extern .shared .align 1024 .b8 smem[];")
L.append(".visible .entry cg(.param .align 64 .b8 tmap[128], .param .u64 pY, .param .u32 ldy4, .param .u32 N)")
L.append(f".maxntid {T}, 1, 1")
L.append("{")
L.append(f"  .reg .b64 a<{R}>; .reg .b64 x<{PF + 1}>; .reg .b64 ww, py, pc, t64, tm; .reg .b32 r<40>; .reg .pred p<8>;")
L.append("  mov.u32 r0, %tid.x; shr.u32 r1, r0, 5; and.b32 r2, r0, 31;")  # r1 warp, r2 lane
L.append(f"  mov.u32 r3, %ctaid.x; mul.lo.u32 r4, r3, {64 * W};")  # n0
L.append("  mov.u32 r5, smem;")
L.append("  setp.ne.u32 p0, r0, 0; @p0 bra INITDONE;")
for s in range(S):
    L.append(f"  mbarrier.init.shared::cta.b64 [r5+{BAR + 8 * s}], 1;")
    L.append(f"  mbarrier.init.shared::cta.b64 [r5+{BAR + 8 * (S + s)}], {W};")
L.append("  fence.mbarrier_init.release.cluster;")
L.append("INITDONE:")
L.append("  bar.sync 0;")
L.append(f"  setp.ne.u32 p1, r1, {W}; @p1 bra CONSUMER;")
# ---------------- producer (runtime loop)
L.append("  setp.ne.u32 p2, r2, 0; @p2 bra DONE;")
L.append("  mov.b64 tm, tmap; cvta.param.u64 tm, tm;")
L.append("  mov.u32 r20, 0;")  # step j
L.append("PLOOP:")
L.append(f"  and.b32 r21, r20, {S - 1}; shr.u32 r22, r20, {LS};")  # s, round
L.append(f"  setp.lt.u32 p3, r20, {S}; @p3 bra PNOWAIT;")
L.append("  sub.u32 r23, r22, 1; and.b32 r23, r23, 1;")
L.append(f"  mad.lo.u32 r24, r21, 8, {BAR + 8 * S}; add.u32 r24, r24, r5;")
L.append("PWE: mbarrier.try_wait.parity.shared::cta.b64 p4, [r24], r23; @!p4 bra PWE;")
L.append("PNOWAIT:")
L.append(f"  mad.lo.u32 r25, r21, 8, {BAR}; add.u32 r25, r25, r5;")
L.append(f"  mbarrier.arrive.expect_tx.shared::cta.b64 _, [r25], {STAGE};")
L.append(f"  mad.lo.u32 r26, r21, {STAGE}, r5;")  # stage base
for b in range(W):
    # chunk = (j + off_b) mod NCH
    L.append(f"  add.u32 r27, r20, {offs[b]}; rem.u32 r27, r27, {NCH}; mul.lo.u32 r27, r27, {KC};")
    L.append(f"  add.u32 r6, r4, {64 * b}; add.u32 r7, r26, {b * BOX};")
    L.append("  cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [r7], [tm, {r6, r27}], [r25];")
L.append(f"  add.u32 r20, r20, 1; setp.lt.u32 p5, r20, {NCH}; @p5 bra PLOOP;")
L.append("  bra DONE;")
# ---------------- consumer
L.append("CONSUMER:")
L.append("  setp.eq.u32 p5, r2, 0;")
L.append("  shl.b32 r11, r2, 1;")
L.append(f"  mul.lo.u32 r9, r1, {BOX}; shl.b32 r10, r2, 3; add.u32 r9, r9, r10; add.u32 r12, r5, r9;")  # warp/lane base
for i in range(R):
    L.append(f"  mov.b64 a{i}, 0;")
L.append("  mov.u32 r30, 0;")  # step
by_chunk = {}
for c, rows in cols:
    by_chunk.setdefault(c // KC, []).append((c, rows))
# dispatch to the warp's start chunk
for w in range(W):
    L.append(f"  setp.eq.u32 p6, r1, {w}; @p6 bra C{offs[w]};")
for j in range(NCH):
    L.append(f"C{j}:")
    L.append(f"  and.b32 r31, r30, {S - 1}; shr.u32 r32, r30, {LS}; and.b32 r32, r32, 1;")
    L.append(f"  mad.lo.u32 r33, r31, 8, {BAR}; add.u32 r33, r33, r5;")
    L.append(f"  mad.lo.u32 r34, r31, {STAGE}, r12;")  # this lane's X base in the stage
    L.append(f"WF{j}: mbarrier.try_wait.parity.shared::cta.b64 p4, [r33], r32; @!p4 bra WF{j};")
    ch = by_chunk.get(j, [])
    xo = [(c % KC) * 256 for c, _ in ch]
    for i in range(min(PF, len(ch))):
        L.append(f"  ld.shared.b64 x{i % (PF + 1)}, [r34+{xo[i]}];")
    for i, (c, rows) in enumerate(ch):
        if i + PF < len(ch):
            L.append(f"  ld.shared.b64 x{(i + PF) % (PF + 1)}, [r34+{xo[i + PF]}];")
        xr = f"x{i % (PF + 1)}"
        for r in rows:
            L.append(f"  mov.b64 ww, {imm2(rng.gauss(0, 0.05))}; fma.rn.f32x2 a{r}, ww, {xr}, a{r};")
    L.append("  bar.warp.sync -1;")
    L.append(f"  @!p5 bra NA{j};")
    L.append(f"  mad.lo.u32 r35, r31, 8, {BAR + 8 * S}; add.u32 r35, r35, r5;")
    L.append("  mbarrier.arrive.shared::cta.b64 _, [r35];")
    L.append(f"NA{j}:")
    L.append(f"  add.u32 r30, r30, 1; setp.eq.u32 p7, r30, {NCH}; @p7 bra EPI;")
L.append("  bra C0;")
L.append("EPI:")
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
