"""Pins for the oracle's block hashing (R2: the paper only says "salted hash
blocks (16 tokens per block)").  The hash is our reading, so the pins are the
published splitmix64 reference outputs for the finaliser and the structural
properties any salted *prefix* hash must have (P:360 radix-tree prefix identity)."""
import numpy as np
import pytest

from oracle import oracle as O

M64 = (1 << 64) - 1


def test_fmix64_matches_published_splitmix64_outputs():
    # splitmix64 reference generator (Vigna, prng.di.unimi.it/splitmix64.c) seeded with 0
    # emits fmix64(k * 0x9E3779B97F4A7C15) for k = 1, 2, 3 ...  Published first outputs:
    expected = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    for k, e in enumerate(expected, start=1):
        assert O.fmix64((k * 0x9E3779B97F4A7C15) & M64) == e


def test_fmix64_is_bijective_on_a_sample(rng):
    xs = rng.integers(0, 2**63, 20000, dtype=np.int64).astype(np.uint64)
    ys = {O.fmix64(int(x)) for x in xs}
    assert len(ys) == len(set(int(x) for x in xs))


def test_partial_tail_never_hashed(rng):
    t = rng.integers(0, 150000, 16 * 5 + 9, dtype=np.int64).astype(np.uint32)
    h = O.chain_hashes(t)
    assert len(h) == 5
    h2 = O.chain_hashes(t[: 16 * 5])
    assert np.array_equal(h, h2)


def test_equal_prefixes_give_equal_chains_and_a_token_change_changes_exactly_the_suffix(rng):
    t = rng.integers(0, 150000, 16 * 12, dtype=np.int64).astype(np.uint32)
    h = O.chain_hashes(t, salt=7)
    for p in [0, 5, 15, 16, 17, 100, 16 * 12 - 1]:
        u = t.copy()
        u[p] ^= np.uint32(1 + (p % 5))
        g = O.chain_hashes(u, salt=7)
        kb = p // 16
        assert np.array_equal(g[:kb], h[:kb]), p
        assert np.all(g[kb:] != h[kb:]), p


def test_salt_changes_every_block(rng):
    t = rng.integers(0, 150000, 16 * 8, dtype=np.int64).astype(np.uint32)
    assert np.all(O.chain_hashes(t, salt=1) != O.chain_hashes(t, salt=2))


def test_every_token_of_a_block_matters(rng):
    t = rng.integers(0, 150000, 16, dtype=np.int64).astype(np.uint32)
    c = O.content_hash(t)
    for i in range(16):
        u = t.copy()
        u[i] += np.uint32(1)
        assert O.content_hash(u) != c


def test_same_content_different_prefix_differs(rng):
    a = rng.integers(0, 150000, 16, dtype=np.int64).astype(np.uint32)
    b = rng.integers(0, 150000, 16, dtype=np.int64).astype(np.uint32)
    c = rng.integers(0, 150000, 16, dtype=np.int64).astype(np.uint32)
    h1 = O.chain_hashes(np.concatenate([a, c]))
    h2 = O.chain_hashes(np.concatenate([b, c]))
    assert h1[1] != h2[1]
    # prefix identity: the block hash of [a] equals the first block of [a, c]
    assert O.chain_hashes(a)[0] == h1[0]


def test_no_collisions_on_a_synthetic_trace():
    import kareto_inputs as ki
    tr = ki.synthetic("chat", R=300, seed=3)
    hs = []
    for r in range(tr.n_requests):
        hs.append(O.chain_hashes(tr.tokens[tr.offsets[r]:tr.offsets[r + 1]]))
    allh = np.concatenate(hs)
    # distinct prefixes == distinct hashes: count distinct token prefixes independently
    prefixes = set()
    for r in range(tr.n_requests):
        seq = tr.tokens[tr.offsets[r]:tr.offsets[r + 1]]
        n = len(seq) // 16
        for k in range(n):
            prefixes.add(hash(seq[: 16 * (k + 1)].tobytes()))
    assert len(np.unique(allh)) == len(prefixes)
