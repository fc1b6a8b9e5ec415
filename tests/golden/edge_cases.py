"""Hand-written planning inputs exercising the branches the reference unit tests
pin (test_graph.cpp, test_scaling.cpp, test_allocation.cpp, test_placement.cpp)
and the outcome classes of SURVEY P6/P12.  Each case is (name, workload text,
topology text, options); expected outputs come from the reference planner
(tests/golden/make_golden.py) and are committed in cases.json.gz.
"""

TOPO8 = "island 0: 0 1 2 3\nisland 1: 4 5 6 7\nbw intra=1e11 inter=2e10\nmem 85899345920\n"
TOPO4 = "island 0: 0 1 2 3\nbw intra=1e11 inter=2e10\nmem 1099511627776\n"


def topo(n, island, mem=85899345920, ids=None):
    ids = ids or list(range(n))
    lines = []
    for i in range(0, n, island):
        lines.append(f"island {i // island}: " + " ".join(str(d) for d in ids[i:i + island]))
    return "\n".join(lines) + f"\nbw intra=1e11 inter=2e10\nmem {mem}\n"


def mod(kind, layers, B=48, tp=1, group=None, param=1000000, w=1.0, c=0.0, act=1000, out=None, seq=1, hidden=1):
    s = f"module {kind} layers={layers} B={B} seq={seq} hidden={hidden} tp={tp}"
    if group:
        s += f" param_group={group}"
    s += f" param_bytes={param} w={w} c={c} act_bytes={act}"
    if out:
        s += f" out_bytes={out}"
    return s + "\n"


def truth(kind, *pieces):
    return "".join(f"truth {kind} piece {lo} {hi} {a} {bc} {bw}\n" for lo, hi, a, bc, bw in pieces)


def cases():
    out = []

    def add(name, w, t, **opt):
        out.append((name, w, t, opt))

    # --- graph shapes (test_graph.cpp:58-248) ---
    w = mod("text-enc", 12, group="g.text") + mod("head-a", 1) + mod("head-b", 1)
    w += truth("text-enc", (1, 1024, 0.01, 0, 0.5)) + truth("head-a", (1, 1024, 0.001, 0, 0.01))
    w += truth("head-b", (1, 1024, 0.002, 0, 0.02))
    w += "task ta flow=text-enc,head-a\ntask tb flow=text-enc,head-b\n"
    add("graph/shared-encoder", w, TOPO8)
    w = mod("solo", 1) + truth("solo", (1, 1024, 0.01, 0, 1.0)) + "task t flow=solo\n"
    add("graph/single-op", w, TOPO8)
    w = mod("a", 3) + mod("b", 4) + truth("a", (1, 1024, 0.0, 0, 1.0)) + truth("b", (1, 1024, 0.01, 0, 0.5))
    w += "task t0 flow=a\ntask t1 flow=b\n"
    add("graph/disjoint", w, TOPO8)
    w = mod("va", 3) + mod("vb", 3) + mod("fuse", 2)
    w += truth("va", (1, 1024, 0.01, 0, 1.0)) + truth("vb", (1, 1024, 0.02, 0, 0.6)) + truth("fuse", (1, 1024, 0, 0, 0.5))
    w += "task t flow=va+vb,fuse\n"
    add("graph/two-towers-fusion", w, TOPO8)
    w = mod("src", 2) + mod("l", 2) + mod("r", 3) + mod("sink", 1)
    for k in ("src", "l", "r", "sink"):
        w += truth(k, (1, 1024, 0.001, 0, 0.3))
    w += "task t flow=src,l+r,sink\n"
    add("graph/diamond", w, TOPO8)
    w = mod("a", 2) + mod("b", 2) + mod("c", 2)
    for k in ("a", "b", "c"):
        w += truth(k, (1, 1024, 0.001, 0, 0.3))
    w += "task t0 flow=a,b,c\ntask t1 flow=a,c\n"
    add("graph/skip-edge", w, TOPO8)
    w = mod("a", 2) + mod("b", 2) + truth("a", (1, 1024, 0, 0, 1)) + truth("b", (1, 1024, 0, 0, 1))
    w += "task t0 flow=a,b\ntask t1 flow=b,a\n"
    add("graph/cycle", w, TOPO8)
    w = mod("a", 1) + truth("a", (1, 1024, 0, 0, 1)) + "task t0 flow=a>a\n"
    add("graph/self-loop", w, TOPO8)
    w = mod("a", 3) + mod("b", 2) + truth("a", (1, 1024, 0, 0, 1)) + truth("b", (1, 1024, 0, 0, 1))
    w += "task t0 flow=a>b\ntask t1 flow=a>b+a>b\ntask t2 flow=a+a,b\n"
    add("graph/duplicate-flows", w, TOPO8)
    # op-id order depends on layers: kind 'enc' vs 'enc.x', 'enc-a'
    w = mod("enc", 12) + mod("enc.x", 3) + mod("enc-a", 2) + mod("enc.1", 2) + mod("z", 1)
    for k in ("enc", "enc.x", "enc-a", "enc.1", "z"):
        w += truth(k, (1, 1024, 0.001, 0, 0.4))
    w += "task t0 flow=enc+enc.x+enc-a+enc.1,z\n"
    add("graph/prefix-kinds", w, TOPO8)
    w = "".join(mod(f"m{i}", 1 + i % 3) for i in range(12))
    w += "".join(truth(f"m{i}", (1, 1024, 0.001 * i, 0, 0.1 + 0.05 * i)) for i in range(12))
    w += "task t0 flow=" + "+".join(f"m{i}" for i in range(12)) + "\n"
    add("graph/ten-plus-metaops", w, topo(16, 8))
    # unused declared module (planner.hpp:69 fits every kind)
    w = mod("used", 2) + mod("unused", 2) + truth("used", (1, 1024, 0, 0, 1)) + truth("unused", (1, 1024, 0, 0, 1))
    w += "task t flow=used\n"
    add("graph/unused-module", w, TOPO8)

    # --- curves (test_scaling.cpp:26-208) ---
    pts = "".join(f"metaop k n={n} config=dp time={0.5 + 8.0 / n!r}\n" for n in range(1, 9))
    w = mod("k", 4, B=840) + pts + "task t flow=k\n"
    add("fit/profile-0.5+8/n", w, TOPO8)
    pts = "".join(f"metaop k n={n} config=dp time=0.25\n" for n in range(1, 9))
    w = mod("k", 4, B=840) + pts + "task t flow=k\n"
    add("fit/flat-profile", w, TOPO8)
    pts = "".join(f"metaop k n={n} config=dp time={(0.1 + 4.0 / n) if n <= 4 else (0.2 + 3.6 / n)!r}\n"
                  for n in range(1, 9))
    w = mod("k", 6, B=840) + pts + "breakpoints k 4\n" + "task t flow=k\n"
    add("fit/two-piece-breakpoint", w, TOPO8)
    pts = "".join(f"metaop k n={n} config=dp time={0.1 + 0.01 * n!r}\n" for n in range(1, 9))
    w = mod("k", 4, B=840) + pts + "task t flow=k\n"
    add("fit/isotonic-increasing", w, TOPO8)
    pts = "".join(f"metaop k n={n} config=dp time={1.0 / n + (0.3 if n == 5 else 0.0)!r}\n" for n in range(1, 9))
    w = mod("k", 4, B=840) + pts + "task t flow=k\n"
    add("fit/isotonic-bump", w, TOPO8)
    w = mod("k", 4, B=840) + "metaop k n=2 config=dp time=1.0\nmetaop k n=2 config=dp time=1.1\n" + "task t flow=k\n"
    add("fit/one-distinct-n", w, TOPO8)
    pts = "".join(f"metaop k n={n} config=dp time={1.0 / n!r}\n" for n in range(1, 5))
    w = mod("k", 4, B=840) + pts + "breakpoints k 6\n" + "task t flow=k\n"
    add("fit/breakpoint-outside-span", w, TOPO8)
    pts = "".join(f"metaop k n={n} config=dp time={1.0 / n!r}\n" for n in range(1, 5))
    w = mod("k", 4, B=840) + pts + "breakpoints k 3 2\n" + "task t flow=k\n"
    add("fit/breakpoints-unsorted", w, TOPO8)
    pts = "".join(f"metaop k n={n} config=dp time={1.0 / n!r}\n" for n in range(1, 5))
    w = mod("k", 4, B=840) + pts + "task t flow=k\n"
    add("fit/profile-nmax-below-N", w, TOPO8)
    w = mod("k", 4, B=840) + truth("k", (1, 1024, -0.5, 0, 0.1)) + "task t flow=k\n"
    add("fit/nonpositive-sample", w, TOPO8)
    pts = "".join(f"metaop k n={n} config=dp time={t}\n" for n, t in [(1, 10), (2, 0.1), (4, 0.1), (8, 0.1)])
    w = mod("k", 4, B=840) + pts + "task t flow=k\n"
    add("fit/degenerate-nonpositive", w, TOPO8)
    w = mod("k", 4) + mod("j", 2) + truth("k", (1, 1024, 0.1, 0, 1)) + "task t flow=k,j\n"
    add("fit/no-source", w, TOPO8)
    w = mod("k", 4) + truth("k", (9, 1024, 0.1, 0, 1)) + "task t flow=k\n"
    add("fit/truth-out-of-range", w, TOPO8)
    w = mod("k", 4) + truth("k", (2, 1024, 0.1, 0, 1)) + "task t flow=k\n"
    add("fit/truth-not-from-1", w, TOPO8)
    w = mod("k", 4) + truth("k", (1, 3, 0.1, 0, 1), (4, 1024, 0.1, 0, 1)) + "task t flow=k\n"
    add("fit/truth-gap", w, TOPO8)
    w = mod("k", 4, w=2.0, c=0.5) + truth("k", (4, 1024, 0.05, 0.1, 0.4), (1, 4, 0.1, 0.1, 0.5)) + "task t flow=k\n"
    add("fit/truth-unsorted-pieces", w, TOPO8)
    w = mod("k", 4, w=2.0, c=0.5) + truth("k", (4, 6, 0.05, 0.1, 0.4), (1, 4, 0.1, 0.1, 0.5), (6, 1024, 0.0, 0.1, 0.5))
    w += "task t flow=k\n"
    add("fit/truth-unsorted-valid", w, TOPO8)
    w = mod("k", 6, w=2.0, c=0.5) + truth("k", (1, 2, 0.1, 0.1, 0.5), (2, 5, 0.12, 0.1, 0.4), (5, 1024, 0.2, 0.1, 0.3))
    w += "task t flow=k\n"
    add("fit/truth-three-pieces", w, topo(16, 8))
    w = mod("k", 6, w=2.0, c=0.5) + truth("k", (1, 2, 0.1, 0.1, 0.5), (2, 5, 0.12, 0.1, 0.4), (5, 1024, 0.2, 0.1, 0.3))
    w += "breakpoints k 1 16 3\ntask t flow=k\n"
    add("fit/breakpoints-filtered-to-empty-then-bad", w, topo(16, 8))

    # --- allocation (test_allocation.cpp) ---
    w = mod("big", 8, B=48, tp=16) + truth("big", (1, 1024, 0.1, 0, 1)) + "task t flow=big\n"
    add("alloc/tp-exceeds", w, TOPO8)
    w = mod("a", 10, B=5040) + mod("b", 20, B=5040)
    w += truth("a", (1, 1024, 0, 0, 8.0)) + truth("b", (1, 1024, 0, 0, 2.0)) + "task t0 flow=a\ntask t1 flow=b\n"
    add("alloc/closed-form-30", w, TOPO4)
    w = mod("a", 7, B=7) + mod("b", 5, B=7) + mod("c", 3, B=7)
    w += truth("a", (1, 1024, 0.5, 0, 1)) + truth("b", (1, 1024, 0.5, 0, 1)) + truth("c", (1, 1024, 0.5, 0, 1))
    w += "task t0 flow=a\ntask t1 flow=b\ntask t2 flow=c\n"
    add("alloc/prime-batches", w, TOPO8)
    w = "".join(mod(f"f{i}", 4, B=12) for i in range(6)) + "".join(truth(f"f{i}", (1, 1024, 0.3, 0, 1e-9)) for i in range(6))
    w += "task t flow=" + "+".join(f"f{i}" for i in range(6)) + "\n"
    add("alloc/flat-curves-repair", w, topo(4, 4))
    w = mod("a", 9, B=48) + mod("b", 5, B=48, tp=2) + mod("c", 3, B=48)
    w += truth("a", (1, 1024, 0.01, 0, 1)) + truth("b", (1, 1024, 0.02, 0, 0.7)) + truth("c", (1, 1024, 0.0, 0, 0.2))
    w += "task t flow=a+b+c\n"
    add("alloc/drop-floor", w, TOPO8, drop_floor=0.2)
    add("alloc/eps-max-iters", w, TOPO8, eps=1e-12, max_iters=7)

    # --- placement (test_placement.cpp) ---
    w = mod("a", 4, B=48, param=10**9, act=10**8) + mod("b", 4, B=48, param=10**9, act=10**8)
    w += truth("a", (1, 1024, 0.01, 0, 1)) + truth("b", (1, 1024, 0.01, 0, 1)) + "task t flow=a,b\n"
    add("place/infeasible-memory", w, topo(2, 2, mem=10**6))
    w = "".join(mod(f"h{i}", 2, B=48, param=3 * 10**8, act=10**7, group="shared" if i % 2 else None) for i in range(6))
    w += "".join(truth(f"h{i}", (1, 1024, 0.01, 0, 0.5 + 0.1 * i)) for i in range(6))
    w += "task t0 flow=h0+h1+h2,h3\ntask t1 flow=h4,h5\n"
    add("place/memory-tight-backtrack", w, topo(8, 4, mem=3 * 10**9))
    add("place/memory-tight-bt0", w, topo(8, 4, mem=3 * 10**9), bt_depth=0)
    add("place/memory-tight-bt-wide", w, topo(8, 4, mem=3 * 10**9), bt_depth=3, bt_branching=4)
    add("place/memory-tight-seq", w, topo(8, 4, mem=3 * 10**9), sequential=1)
    w = mod("p", 3, B=48, group="m1", param=5 * 10**8, act=10**6) + mod("q", 3, B=48, param=5 * 10**8, act=10**6)
    w += mod("r", 2, B=48, group="m0", param=10**8)
    w += truth("p", (1, 1024, 0.01, 0, 1)) + truth("q", (1, 1024, 0.01, 0, 1)) + truth("r", (1, 1024, 0.01, 0, 1))
    w += "task t flow=p+q,r\n"
    add("place/group-named-like-entity", w, topo(8, 4, mem=4 * 10**9))
    w = mod("x", 6, B=48, act=10**7, out=10**5) + mod("y", 4, B=48, act=10**7) + mod("z", 2, B=48, act=10**6)
    w += truth("x", (1, 1024, 0.01, 0, 1)) + truth("y", (1, 1024, 0.02, 0, 0.3)) + truth("z", (1, 1024, 0, 0, 0.1))
    w += "task t0 flow=x,y,z\ntask t1 flow=x,z\n"
    add("place/odd-device-ids", w, topo(8, 4, ids=[3, 9, 11, 40, 5, 17, 100, 2]))
    add("place/single-device", w, topo(1, 1))
    pts = "".join(f"metaop {k} n=1 config=dp time=0.5\nmetaop {k} n=2 config=dp time=0.3\n" for k in "xyz")
    w1 = mod("x", 2, B=48) + mod("y", 2, B=48) + mod("z", 2, B=48) + pts + "task t0 flow=x,y,z\n"
    add("place/single-device-profiles", w1, topo(1, 1))
    add("place/sequential-ablation", w, topo(8, 4), sequential=1)
    add("place/uneven-islands", w,
        "island 0: 0 1 2\nisland 1: 3 4 5 6 7\nisland 2: 8\nbw intra=1e11 inter=1e10\nmem 85899345920\n")
    w = "".join(mod(f"e{i:02d}", 1 + i % 4, B=6720, act=10**6 * (1 + i % 5), out=10**4 * (1 + i % 3),
                    group=f"g{i % 7}", param=10**7 * (1 + i % 3)) for i in range(20))
    w += "".join(truth(f"e{i:02d}", (1, 8, 0.01, 0.0, 0.2 + 0.03 * i), (8, 1024, 0.012, 0.0, 0.21 + 0.03 * i))
                 for i in range(20))
    w += "task a flow=" + "+".join(f"e{i:02d}" for i in range(0, 10)) + ",e19\n"
    w += "task b flow=" + "+".join(f"e{i:02d}" for i in range(10, 19)) + ",e19\n"
    add("place/max-devices-64", w, topo(64, 8))
    add("place/max-devices-64-seq", w, topo(64, 8), sequential=1)
    add("options/grad-mult", w, topo(32, 8), grad_mult=0.5)
    add("options/noise", w, topo(32, 8), synth_noise=0.05, synth_seed=11)
    return out
