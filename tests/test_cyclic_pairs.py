"""Host-side check of the pair enumeration behind the rolled 5x5 exact exp/log
window (csrc/vf_window.cuh, el_window_s1): for odd N the pairs
{k, (k + d) mod N}, d = 1 .. (N - 1) / 2, are every unordered pair of the
window once (each aggregate sums the criterion over all other
samples), and after (N - 1) / 2 one-position rotations the rotating partial
aggregate in slot k belongs to sample (k + (N - 1) / 2) mod N."""
import itertools

import pytest


@pytest.mark.parametrize("n", [9, 25, 49])
def test_cyclic_offsets_enumerate_every_pair_once(n):
    seen = [frozenset((k, (k + d) % n)) for d in range(1, (n - 1) // 2 + 1) for k in range(n)]
    assert len(seen) == len(set(seen)) == n * (n - 1) // 2
    assert set(seen) == {frozenset(p) for p in itertools.combinations(range(n), 2)}


@pytest.mark.parametrize("n", [9, 25])
def test_rotating_registers_return_to_their_samples(n):
    # the kernel's loop, with sets of partner indices in place of float sums
    wb = list(range(n))
    ra = [set() for _ in range(n)]
    rb = [set() for _ in range(n)]
    for d in range(1, (n - 1) // 2 + 1):
        wb = wb[1:] + wb[:1]
        rb = rb[1:] + rb[:1]
        for k in range(n):
            assert wb[k] == (k + d) % n
            ra[k].add(wb[k])          # sample k meets sample wb[k]
            rb[k].add(k)              # and sample wb[k] meets sample k
    for k in range(n):
        ra[(k + (n - 1) // 2) % n] |= rb[k]
    for i in range(n):
        assert ra[i] == set(range(n)) - {i}
