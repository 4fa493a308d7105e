"""Host logic of the gathered-parameter slots (CPU): the 2-slot ring, the reuse cache
(param_cache=K) and the head's slot, simulated over one step's fetch / use / release
sequence exactly as GPTZeroEngine.step issues it."""

import types

import pytest

from paper_2104_07857_b200.gpt import GPTZeroEngine


def _slot(K, i, nb):
    return GPTZeroEngine._pslot(types.SimpleNamespace(K=K), i, nb)


@pytest.mark.parametrize("nb", [1, 2, 3, 5, 24, 87])
@pytest.mark.parametrize("K", [0, 1, 2, 11, 40, 86])
def test_slot_sequence_never_overwrites_a_live_bucket(nb, K):
    K = min(K, max(0, nb - 1))
    HEAD = nb
    content = {}                      # slot -> bucket it holds
    fetches = 0

    def fetch(b):
        nonlocal fetches
        fetches += 1
        content[_slot(K, b, nb)] = b

    def use(b):
        assert content.get(_slot(K, b, nb)) == b, (b, content)

    # forward: block i+1 (or the head) is fetched while block i computes; the ring slot
    # it lands in was last read by block i-1 (finished)
    fetch(0)
    for i in range(nb):
        fetch(i + 1 if i + 1 < nb else HEAD)
        use(i)
        if i + 1 < nb:                # the bucket being fetched must not evict block i
            assert _slot(K, i + 1, nb) != _slot(K, i, nb)
    assert _slot(K, HEAD, nb) != _slot(K, nb - 1, nb)
    use(HEAD)
    # backward: blocks nb-1 .. 0; only blocks below nb-1-K are fetched again
    for j in range(nb - 1, -1, -1):
        use(j)
        if 0 <= j - 1 < nb - 1 - K:
            assert _slot(K, j - 1, nb) != _slot(K, j, nb)
            fetch(j - 1)
    assert fetches == (nb + 1) + max(0, nb - 1 - K)
    cache = {_slot(K, i, nb) for i in range(nb - K, nb)} if K else set()
    assert len(cache) == K and all(s >= 2 for s in cache)
