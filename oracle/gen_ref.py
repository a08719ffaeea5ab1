"""CPU restatement of libb2's seeded input generator (kernels.cu
gen_normal_kernel / gen_tokens_kernel) — TEST INFRASTRUCTURE ONLY.

element i of stream `seed`: h = splitmix64(seed * 0xD1B54A32D192ED03 + i);
normal = sqrt(-2 ln u1) cos(2 pi u2) with u1 = ((h >> 40) + 1) / 2^24,
u2 = ((h >> 16) & 0xFFFFFF) / 2^24; token = ((h >> 32) * vocab) >> 32.
"""
import numpy as np

M64 = (1 << 64) - 1


def splitmix64(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _hash(n, seed):
    with np.errstate(over="ignore"):
        base = np.uint64((seed * 0xD1B54A32D192ED03) & M64)
        return splitmix64(base + np.arange(n, dtype=np.uint64))


def normal(n, seed):
    h = _hash(n, seed)
    u1 = ((h >> np.uint64(40)).astype(np.float64) + 1.0) / 16777216.0
    u2 = ((h >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.float64) / 16777216.0
    return (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).astype(np.float32)


def tokens(n, vocab, seed):
    h = _hash(n, seed)
    return (((h >> np.uint64(32)) * np.uint64(vocab)) >> np.uint64(32)).astype(np.int64)


def plan_tokens(batch, seq, vocab, seed, masked):
    """The token input b2_gen_input writes for a plan: per sample [ids(seq)]
    or, for attention-mask plans, [ids(seq), ones(seq)]; id j of sample b is
    stream element b * seq + j either way (kernels.cu gen_tokens_kernel)."""
    ids = tokens(batch * seq, vocab, seed).reshape(batch, seq)
    if not masked:
        return ids.reshape(-1)
    return np.concatenate([ids, np.ones((batch, seq), np.int64)], 1).reshape(-1)
