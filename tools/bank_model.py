"""Shared-memory bank model of the row kernels' access patterns (dev tool).

Counts wavefronts per warp-instruction phase the way the L1 serves 64-bit
shared accesses (two half-warp phases of 16 lanes, 16 bank pairs; a phase
costs the largest number of distinct addresses sharing a bank pair) for:
  * K3 (N = 512): the radix-16 exchange puts/gets and the row-separation loop,
    XOR-swizzled layout (stride 258) vs padded layout (addr = i + i/16),
  * K5 (N = 512): the stride-3 reads of the TMA-staged Y rows and the radix-3
    combine, row-major vs q-major transform order,
  * K5 (every N): the stride-3 bin reads of the blocked, row-permuted Y layout
    K4 stores (pipeline.h y_at / y_swz), and that the permutation is one.
usage: python tools/bank_model.py [k5y]"""
from collections import Counter


def cost(addrs):
    addrs = set(a for a in addrs if a is not None)
    return max(Counter(a % 16 for a in addrs).values()) if addrs else 0


def xor_at(i):
    return (i & ~15) | ((i & 15) ^ ((i >> 4) & 15))


def pad_at(i):
    return i + (i >> 4)


def k3(at, stride, K=256, T=16, TH=384, ROWS=8, H=384):
    O = (3 * stride) % 16
    KB = 16 if O == 0 else min(O & -O, 16)
    R = 16 // KB
    RG = ROWS // R
    KSTEP = TH // ROWS
    tot, ideal = Counter(), Counter()

    def addr(tr, i):
        return tr * stride + at(i)

    def sep_map(tid):
        g, hl = tid >> 4, tid & 15
        return (g % RG) * R + hl // KB, (g // RG) * KB + hl % KB

    for w in range(TH // 32):
        for hw in (0, 1):
            lanes = range(w * 32 + 16 * hw, w * 32 + 16 * hw + 16)
            for r in range(16):
                tot["exchange"] += cost(addr(t // T, 16 * (t % T) + r) for t in lanes)
                ideal["exchange"] += 1
            for m in range(16):
                tot["exchange"] += cost(addr(t // T, t % T + 16 * m) for t in lanes)
                ideal["exchange"] += 1
            for loop in range(3):
                for it in range(10):
                    a1, a2 = [], []
                    for tid in lanes:
                        ol, kk = sep_map(tid)
                        k = kk + it * KSTEP
                        if loop == 0 and k <= K // 2:
                            a1.append(addr(3 * ol, k)); a2.append(addr(3 * ol, (K - k) & (K - 1)))
                        if loop == 1 and 3 * k + 1 <= H:
                            a1.append(addr(3 * ol + 1, k)); a2.append(addr(3 * ol + 2, K - 1 - k))
                        if loop == 2 and 3 * k + 2 <= H:
                            a1.append(addr(3 * ol + 2, k)); a2.append(addr(3 * ol + 1, K - 1 - k))
                    for a in (a1, a2):
                        if a:
                            tot["separation"] += cost(a); ideal["separation"] += 1
    return dict(tot), dict(ideal)


def k5(qmajor, at=xor_at, stride=136, T=8, ROWS=8, TH=192, RPS=392, H=384):
    tot, ideal = Counter(), Counter()

    def rq(tid):
        tr, t = tid // T, tid % T
        return (tr, t, tr % ROWS, tr // ROWS) if qmajor else (tr, t, tr // 3, tr % 3)

    for w in range(TH // 32):
        for hw in (0, 1):
            lanes = range(w * 32 + 16 * hw, w * 32 + 16 * hw + 16)
            for m in range(16):
                for which in (0, 1):
                    a = []
                    for tid in lanes:
                        tr, t, rl, q = rq(tid)
                        k = 3 * (t + 8 * m) + q
                        a.append(rl * RPS + (k if which == 0 else H - k))
                    tot["y_reads"] += cost(a); ideal["y_reads"] += 1
            for j in range(6):
                for qq in range(3):
                    a = []
                    for tid in lanes:
                        tr, t, rl, q = rq(tid)
                        m = q + 3 * j
                        if m < 16:
                            trq = qq * ROWS + rl if qmajor else 3 * rl + qq
                            a.append(trq * stride + at(t + m * T))
                    if a:
                        tot["combine"] += cost(a); ideal["combine"] += 1
    return dict(tot), dict(ideal)


def y_swz(rb, k):  # pipeline.h
    return (rb // 4) * ((k >> (0 if rb >= 16 else (1 if rb == 8 else 2))) & 3)


def k5y(N):
    """Y[i][k] at k * RB + (rl ^ y_swz(RB, k)) inside the CTA's block; q-major K5."""
    K2, H = N // 4, 3 * N // 4
    T = K2 // 16
    RB = min(4096 // N, N)
    TH = 3 * RB * T
    for k in range(H + 1):
        assert sorted(r ^ y_swz(RB, k) for r in range(RB)) == list(range(RB))
    tot = ideal = 0
    for w in range(TH // 32):
        for m in range(16):
            for mirror in (False, True):
                for h in range(2):
                    a = []
                    for lane in range(16 * h, 16 * h + 16):
                        tr, t = divmod(w * 32 + lane, T)
                        rl, q = tr % RB, tr // RB
                        k = 3 * (t + m * T) + q
                        k = H - k if mirror else k
                        a.append(k * RB + (rl ^ y_swz(RB, k)))
                    tot += cost(a)
                    ideal += 1
    return tot, ideal


if __name__ == "__main__":
    import sys
    if sys.argv[1:] == ["k5y"]:
        for n in (64, 128, 256, 512, 1024):
            print(f"K5 blocked Y, N={n}: wavefronts {k5y(n)[0]} (conflict-free: {k5y(n)[1]})")
        sys.exit(0)
    print("K3 XOR layout, stride 258:", k3(xor_at, 258))
    print("K3 padded layout, stride 274:", k3(pad_at, 274))
    print("K3 N=1024 XOR layout, stride 524:", k3(xor_at, 524, K=512, T=32, TH=384, ROWS=4, H=768))
    print("K3 N=1024 padded layout, stride 556:", k3(pad_at, 556, K=512, T=32, TH=384, ROWS=4, H=768))
    print("K5 row-major:", k5(False))
    print("K5 q-major:", k5(True))
    print("K5 q-major, padded layout (stride 136):", k5(True, pad_at, 136))
