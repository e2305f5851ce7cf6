"""Generate and check the 24-key sorting network of median_tiled_kernel
(Batcher's odd-even merge sort for 32 inputs, comparators touching inputs
24..31 removed).  Prints the flat pair list used as kMedNet in stages.cu."""
import itertools
import random


def batcher_pairs(n=32, keep=24):
    pairs = []
    p = 1
    while p < n:
        k = p
        while k >= 1:
            j = k % p
            while j + k < n:
                for i in range(min(k, n - j - k)):
                    if (i + j) // (2 * p) == (i + j + k) // (2 * p):
                        a, b = i + j, i + j + k
                        if a < keep and b < keep:
                            pairs.append((a, b))
                j += 2 * k
            k //= 2
        p *= 2
    return pairs


def check(pairs, keep=24, trials=20000):
    for _ in range(trials):
        v = [random.randint(0, 40) for _ in range(keep)]
        w = list(v)
        for a, b in pairs:
            if w[a] > w[b]:
                w[a], w[b] = w[b], w[a]
        assert w == sorted(v)


if __name__ == "__main__":
    pr = batcher_pairs()
    check(pr)
    print(len(pr))
    print(",".join(str(x) for x in itertools.chain(*pr)))
