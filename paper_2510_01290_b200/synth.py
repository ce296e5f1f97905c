"""Host-side helpers of the synthetic workload (csrc/synth.h mirrored in Python):
scripted thought labels per sequence and refresh interval."""
from __future__ import annotations

M64 = (1 << 64) - 1


def mix64(a: int, b: int) -> int:
    """splitmix64 finaliser of a + golden * (b + 1) (thinkv::Rng::mix, rng.hpp:56-61)."""
    z = (a + 0x9E3779B97F4A7C15 * (b + 1)) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


ROLE_LABEL = 7


def band(seed: int, seq: int, interval: int, num_thoughts: int, pT_permille: int) -> int:
    """tkv_synth_band: T with probability pT/1000, else the other bands uniformly."""
    h = mix64(mix64(seed, ROLE_LABEL), mix64(seq, interval))
    if num_thoughts < 3:
        return (h >> 20) % num_thoughts
    if h % 1000 < pT_permille:
        return num_thoughts - 1
    return (h >> 20) % (num_thoughts - 1)


def band_script(seed: int, num_seqs: int, intervals: int, num_thoughts: int, pT_permille: int):
    return [[band(seed, s, i, num_thoughts, pT_permille) for i in range(intervals)] for s in range(num_seqs)]
