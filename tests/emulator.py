"""TEST INFRASTRUCTURE: numpy replay of the fused gate-block kernel's semantics
(paper_2409_14697_b200/csrc/engine/block_pass.cu) over the pass programs the
host scheduler emits (qk_debug_compile_block).  Lets the CPU suite check the
scheduler (register maps, deferred factors, X relabels, exchanges, tiles)
against the oracle without a GPU.  Never used by the product."""
import numpy as np

OPS = ["MAT1", "H", "CX", "DIAG1_R", "DIAG2_RR", "CPHASE_RR", "PEND_R", "PEND_RT", "SCAL", "SCAL_T",
       "SCAL_TT", "FLUSH_SLOT", "FLUSH", "DTABLE", "DENSE", "EXCHANGE", "SCAL_TAB", "PEND_TAB", "SCAL_CTA",
       "PEND_CTA", "SCAL_TCTA", "FLUSH_SLOT_G", "RESET", "CX_PEND", "CCX"]


def pext8(t, m):
    r = np.zeros_like(t)
    i = 0
    for j in range(16):
        if (m >> j) & 1:
            r |= ((t >> j) & 1) << i
            i += 1
    return r


def swz(u):
    return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12)) & 7)


def run_steps(state: np.ndarray, n: int, prog: dict) -> None:
    """Apply the compiled steps to `state` (complex128, 2^n) in place."""
    g = np.array(prog["gtab"], dtype=np.float64)
    gt = g[0::2] + 1j * g[1::2]
    for st in prog["steps"]:
        if st["kind"] == 0:
            _run_pass(state, n, st, gt)
        elif st["kind"] == 1:
            _dense_group(state, n, st, gt)
        else:
            _diag_table(state, n, st, gt)


def _dense_group(state, n, st, gt):
    k, tg = st["k"], st["targets"]
    dim = 1 << k
    M = gt[st["mat"]:st["mat"] + dim * dim].reshape(dim, dim)
    off = np.zeros(dim, dtype=np.int64)
    for s in range(dim):
        for j in range(k):
            off[s] |= ((s >> (k - 1 - j)) & 1) << tg[j]
    mask = sum(1 << t for t in tg)
    bases = np.array([i for i in range(1 << n) if not (i & mask)], dtype=np.int64)
    idx = bases[:, None] | off[None, :]
    state[idx] = (M @ state[idx].T).T


def _diag_table(state, n, st, gt):
    k, tg = st["k"], st["targets"]
    i = np.arange(1 << n)
    sub = np.zeros_like(i)
    for j in range(k):
        sub |= ((i >> tg[j]) & 1) << (k - 1 - j)
    state *= gt[st["mat"] + sub]


def _run_pass(state, n, P, gt):
    ct, rb = P["ct"], P["rb"]
    na, nt = 1 << rb, 1 << (ct - rb)
    coef = np.array(P["coef"][0::2]) + 1j * np.array(P["coef"][1::2])
    contrib = P["contrib"]
    tp = P["tile_phys"]
    tid = np.arange(nt)
    s_idx = np.arange(na)

    def bit(x, j):
        return (x >> j) & 1

    def gaddr(m, xm):
        off = np.zeros(nt, dtype=np.int64)
        for j in range(ct - rb):
            off |= bit(tid, j).astype(np.int64) << tp[m[rb + j]]
        so = np.zeros(na, dtype=np.int64)
        for kk in range(rb):
            so |= bit(s_idx, kk).astype(np.int64) << tp[m[kk]]
        x = 0
        for j in range(ct):
            if (xm >> j) & 1:
                x |= 1 << tp[j]
        return (off[:, None] | so[None, :]) ^ x

    def taddr(m, xm):
        u = np.zeros(nt, dtype=np.int64)
        for j in range(ct - rb):
            u |= bit(tid, j).astype(np.int64) << m[rb + j]
        us = np.zeros(na, dtype=np.int64)
        for kk in range(rb):
            us |= bit(s_idx, kk).astype(np.int64) << m[kk]
        return swz((u[:, None] | us[None, :]) ^ xm)

    tile_mask = sum(1 << p for p in tp)
    others = [b for b in range(n) if not (tile_mask >> b) & 1]
    for cta in range(1 << (n - ct)):
        base = 0
        for j, b in enumerate(others):
            base |= ((cta >> j) & 1) << b
        addr = base | gaddr(P["map_in"][0], 0)
        a = state[addr].copy()  # (nt, na)
        F = []
        for f in range(P.get("ncta", 0)):
            acc = 1 + 0j
            for (b1, b2, c) in P["cta_terms"][(P["cta_end"][f - 1] if f else 0):P["cta_end"][f]]:
                if b1 == 255 or ((base >> b1) & (base >> b2) & 1):
                    acc *= coef[c]
            F.append(acc)
        Pt = np.ones(nt, dtype=np.complex128)
        R = np.ones((nt, rb), dtype=np.complex128)
        sm = np.zeros(1 << ct, dtype=np.complex128)
        for (typ, oa, ob, ok, oc, oc16, ox16) in P["ops"]:
            name = OPS[typ]
            if name == "EXCHANGE":
                sm[taddr(P["map_out"][oc - 1], P["xmask_out"][oc - 1])] = a
                a = sm[taddr(P["map_in"][oc], 0)].copy()
            elif name == "H":
                lo = s_idx[(s_idx >> oa) & 1 == 0]
                hi = lo | (1 << oa)
                x, y = a[:, lo].copy(), a[:, hi].copy()
                a[:, lo], a[:, hi] = x + y, x - y
            elif name == "MAT1":
                m = coef[oc:oc + 4]
                lo = s_idx[(s_idx >> oa) & 1 == 0]
                hi = lo | (1 << oa)
                x, y = a[:, lo].copy(), a[:, hi].copy()
                a[:, lo], a[:, hi] = m[0] * x + m[1] * y, m[2] * x + m[3] * y
            elif name == "CX":
                pol = (ok >> 1) & 1
                lo = s_idx[(s_idx >> oa) & 1 == 0]
                hi = lo | (1 << oa)
                if ok & 4:  # control outside the tile: a bit of the CTA's base index
                    cond = np.full((nt, len(lo)), bool((base >> ob) & 1))
                elif ok & 1:
                    cond = ((bit(tid, ob) ^ pol) == 1)[:, None] & np.ones(len(lo), bool)[None, :]
                else:
                    cond = np.broadcast_to(((bit(lo, ob) ^ pol) == 1)[None, :], (nt, len(lo)))
                x, y = a[:, lo].copy(), a[:, hi].copy()
                a[:, lo] = np.where(cond, y, x)
                a[:, hi] = np.where(cond, x, y)
            elif name == "CCX":
                lo = s_idx[(s_idx >> oa) & 1 == 0]
                hi = lo | (1 << oa)
                cond = np.ones((nt, len(lo)), bool)
                for (thr, idx, pol, cta) in (((ok & 1), ob, (ok >> 1) & 1, (ok >> 4) & 1),
                                             ((ok >> 2) & 1, oc, (ok >> 3) & 1, (ok >> 5) & 1)):
                    if cta:
                        cond &= bool((base >> idx) & 1)
                    elif thr:
                        cond &= ((bit(tid, idx) ^ pol) == 1)[:, None]
                    else:
                        cond &= ((bit(lo, idx) ^ pol) == 1)[None, :]
                x, y = a[:, lo].copy(), a[:, hi].copy()
                a[:, lo] = np.where(cond, y, x)
                a[:, hi] = np.where(cond, x, y)
            elif name == "DIAG1_R":
                a *= np.where(bit(s_idx, oa) == 1, coef[oc + 1], coef[oc])[None, :]
            elif name == "DIAG2_RR":
                a *= coef[oc + 2 * bit(s_idx, oa) + bit(s_idx, ob)][None, :]
            elif name == "CPHASE_RR":
                sel = (2 * bit(s_idx, oa) + bit(s_idx, ob)) == ok
                a[:, sel] *= coef[oc]
            elif name == "PEND_R":
                R[:, oa] *= coef[oc]
            elif name == "PEND_RT":
                R[:, oa] *= coef[oc + bit(tid, ob)]
            elif name == "SCAL_TAB":
                Pt *= gt[oc + pext8(tid, ox16)]
            elif name == "PEND_TAB":
                R[:, oa] *= gt[oc + pext8(tid, ox16)]
            elif name == "RESET":
                Pt[:] = 1
                R[:] = 1
            elif name == "FLUSH_SLOT_G":
                bits = [kk for kk in range(rb) if (ob >> kk) & 1]
                for sv in range(na):
                    if (sv >> oa) & 1:
                        j = sum(((sv >> b) & 1) << q for q, b in enumerate(bits))
                        a[:, sv] *= R[:, oa] * coef[oc + j]
                R[:, oa] = 1
            elif name == "CX_PEND":
                act = (bit(tid, ob) ^ ((ok >> 1) & 1)) == 1
                Pt = np.where(act, Pt * R[:, oa], Pt)
                R[:, oa] = np.where(act, 1 / R[:, oa], R[:, oa])
            elif name == "SCAL_CTA":
                Pt *= F[oc]
            elif name == "PEND_CTA":
                R[:, oa] *= F[oc]
            elif name == "SCAL_TCTA":
                Pt *= np.where(bit(tid, ob) == 1, F[oc], 1)
            elif name == "SCAL":
                Pt *= coef[oc]
            elif name == "SCAL_T":
                Pt *= coef[oc + bit(tid, oa)]
            elif name == "SCAL_TT":
                Pt *= coef[oc + 2 * bit(tid, oa) + bit(tid, ob)]
            elif name == "FLUSH_SLOT":
                sel = bit(s_idx, oa) == 1
                a[:, sel] *= R[:, oa][:, None]
                R[:, oa] = 1
            elif name == "FLUSH":
                f = Pt * coef[oc].real
                a *= f[:, None]
                for kk in range(rb):
                    sel = bit(s_idx, kk) == 1
                    a[:, sel] *= R[:, kk][:, None]
                if oc16:
                    a *= coef[oc16 - 1:oc16 - 1 + na][None, :]
                R[:] = 1
                Pt[:] = 1
            elif name == "DTABLE":
                cb = contrib[oc16:oc16 + ct]
                sub = np.zeros(nt, dtype=np.int64)
                for j in range(rb, ct):
                    sub |= np.where(bit(tid, j - rb) == 1, cb[j], 0)
                for j in range(contrib[oc16 + ct]):
                    if (base >> contrib[oc16 + ct + 1 + 2 * j]) & 1:
                        sub |= contrib[oc16 + ct + 2 + 2 * j]
                sr = np.zeros(na, dtype=np.int64)
                for kk in range(rb):
                    sr |= np.where(bit(s_idx, kk) == 1, cb[kk], 0)
                a *= gt[oc + ((sub[:, None] | sr[None, :]) ^ ox16)]
            elif name == "DENSE":
                d = 1 << ok
                M = gt[oc:oc + d * d].reshape(d, d)
                for grp in range(na // d):
                    blk = a[:, grp * d:(grp + 1) * d].copy()
                    a[:, grp * d:(grp + 1) * d] = blk @ M.T
            else:
                raise ValueError(name)
        state[base | gaddr(P["map_out"][-1], P["xmask_out"][-1])] = a
