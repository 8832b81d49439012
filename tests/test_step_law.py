"""The interior-node fast path of the walk engine's MicroWalk step
(walk.cu mw_step, Philox mode): at a node whose six alphas are all 1/2 the
reference's f64 scan (microwalk.cpp:111-124: sum of alphas, in-order partial
sums, first d with target < acc_d) is replaced by dir = floor(6w / 2^32) of
the step's 32-bit word w, except for the words flagged as possible ties
((w * 6) mod 2^32 >= 0xFFFFFFFA), which keep the exact scan.  This checks the
claim exhaustively around each of the five f64 thresholds and on random
words, with Python floats (IEEE binary64, the device's arithmetic)."""
import random

TIE = 0xFFFFFFFA


def scan_dir(x53):
    # the device's general path: sum of six 1/2 alphas, target = x*2^-53*sum
    acc, s = [], 0.0
    for _ in range(6):
        s += 0.5
        acc.append(s)
    target = float(x53) * 2.0 ** -53 * s
    return sum(1 for d in range(5) if acc[d] <= target)


def threshold(k):
    """smallest 53-bit x whose scan direction is >= k"""
    lo, hi = 0, (1 << 53) - 1
    while lo < hi:
        mid = (lo + hi) // 2
        if scan_dir(mid) >= k:
            hi = mid
        else:
            lo = mid + 1
    return lo


def fast(w):
    return (w * 6) >> 32, ((w * 6) & 0xFFFFFFFF) >= TIE


def check_word(w):
    d, tie = fast(w)
    lo, hi = scan_dir(w << 21), scan_dir((w << 21) | 0x1FFFFF)
    if lo != hi:
        assert tie, f"word {w:#x} straddles a threshold but is not flagged"
    elif not tie:
        assert d == lo, f"word {w:#x}: fast {d}, scan {lo}"


def test_interior_fast_path_around_thresholds():
    for k in range(1, 6):
        x = threshold(k)
        w0 = x >> 21
        for w in range(max(0, w0 - 64), min(1 << 32, w0 + 65)):
            check_word(w)


def test_interior_fast_path_random_words():
    rnd = random.Random(5)
    for _ in range(20000):
        check_word(rnd.getrandbits(32))
    for w in (0, 1, (1 << 32) - 1, 1 << 31, (1 << 31) - 1):
        check_word(w)


def test_tie_words_are_rare():
    # at most 6 flagged words per multiple of 2^32 in [0, 6 * 2^32)
    flagged = sum(1 for w in range(0, 1 << 32, 1 << 12) if fast(w)[1])
    assert flagged <= 6
