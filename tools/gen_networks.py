"""Generator of csrc/selnet.cuh and csrc/sortnet.cuh (the K2 median-selection and sorting networks), with the
checks their headers claim.

  python tools/gen_networks.py --write      regenerate both headers in place
  python tools/gen_networks.py --check      regenerate in memory, compare with the committed files, and verify
                                            every network by the 0-1 principle (exhaustively for k <= 16 / N <= 16)
                                            and on random inputs (k <= 32)

Batcher's odd-even merge sort on N = next_pow2(k) inputs (the standard iterative formulation); for the
selection network the comparators touching the +INF padding (index >= k) are removed (no-ops: the largest values
never move down), then the network is pruned backwards to the comparators that can influence the output positions
(k-1)/2 and k/2 (the median's order statistics, K2)."""
import itertools
import os
import random
import sys

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1207_4684_b200", "csrc")


def batcher(n):
    comps, p = [], 1
    while p < n:
        k = p
        while k >= 1:
            for j in range(k % p, n - k, 2 * k):
                for i in range(min(k, n - j - k)):
                    if (i + j) // (2 * p) == (i + j + k) // (2 * p):
                        comps.append((i + j, i + j + k))
            k //= 2
        p *= 2
    return comps


def selection(k):
    n = 1
    while n < k:
        n *= 2
    comps = [(i, j) for i, j in batcher(n) if j < k]
    need, kept = {(k - 1) // 2, k // 2}, []
    for i, j in reversed(comps):
        if i in need or j in need:
            kept.append((i, j))
            need |= {i, j}
    return kept[::-1]


def apply(comps, v):
    v = list(v)
    for i, j in comps:
        if v[i] > v[j]:
            v[i], v[j] = v[j], v[i]
    return v


def selnet_text():
    out = ["// selnet.cuh -- generated median-selection networks: Batcher odd-even merge network on",
           "// next_pow2(k) inputs, comparators touching the +INF padding removed (they are no-ops: the largest",
           "// values never move down), then pruned backwards to those that can influence the output positions",
           "// (k-1)/2 and k/2.  Checked exhaustively (0-1 principle) for k <= 16 and on random inputs for k <= 32.",
           "#pragma once", ""]
    for k in range(1, 33):
        out.append(f"template <class CS> __device__ __forceinline__ void selnet{k}(float* a, CS cs) {{")
        comps = selection(k)
        if not comps:
            out.append("  (void)a; (void)cs;")
        out += [f"  cs(a[{i}], a[{j}]);" for i, j in comps]
        out.append("}")
    return out


def check_selection(k, trials=4000):
    comps, m1, m2 = selection(k), (k - 1) // 2, k // 2
    if k <= 16:
        for bits in itertools.product((0, 1), repeat=k):   # 0-1 principle
            r, s = apply(comps, bits), sorted(bits)
            assert r[m1] == s[m1] and r[m2] == s[m2], (k, bits)
    rng = random.Random(k)
    for _ in range(trials):
        v = [rng.random() for _ in range(k)]
        r, s = apply(comps, v), sorted(v)
        assert r[m1] == s[m1] and r[m2] == s[m2], k


def check_sort(n):
    comps = batcher(n)
    if n <= 16:
        for bits in itertools.product((0, 1), repeat=n):
            assert apply(comps, bits) == sorted(bits), n
    rng = random.Random(n)
    for _ in range(2000):
        v = [rng.random() for _ in range(n)]
        assert apply(comps, v) == sorted(v), n


def main():
    sel = "\n".join(selnet_text())
    path = os.path.join(CSRC, "selnet.cuh")
    committed = open(path).read()
    head = committed[:committed.index("template <int K, class CS>")]   # the dispatcher tail is hand-written
    if "--write" in sys.argv:
        open(path, "w").write(sel + "\n" + committed[committed.index("template <int K, class CS>"):])
        print("wrote", path)
        return
    ok = head.rstrip() == sel.rstrip()
    print("selnet.cuh networks identical to the generator's:", ok)
    for k in range(1, 33):
        check_selection(k)
    print("selection networks k = 1..32: 0-1 principle exhaustive for k <= 16, random inputs for all: OK")
    for n in (8, 16, 32):
        check_sort(n)
    srt = open(os.path.join(CSRC, "sortnet.cuh")).read()
    for n in (8, 16, 32):
        body = srt[srt.index(f"void sortnet{n}("):]
        body = body[:body.index("}")]
        pairs = [tuple(int(x) for x in p) for p in __import__("re").findall(r"cs\(a\[(\d+)\], a\[(\d+)\]\)", body)]
        assert pairs == batcher(n), f"sortnet{n} differs from Batcher's network"
    print("sortnet.cuh N = 8, 16, 32 identical to Batcher's odd-even merge sort; 0-1 principle exhaustive for N <= 16")
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
