"""The stream-K ownership arithmetic the deferred split-K consumers rely on
(csrc/hx_common.cuh: sk_start, sk_owner, sk_tile), restated in numpy and
checked against its definition: CTA c owns units [c*U/G, (c+1)*U/G); the owner
of unit u is the largest c with sk_start(c) <= u, computed in one division as
min(G-1, ((u+1)*G - 1) // U); a tile's first contributor keeps slot 2c or 2c+1
and every later contributor begins inside the tile (slot 2c). CPU only."""

import numpy as np
import pytest


def sk_start(c, units, G):
    return (c * units) // G


def owner_closed(u, units, G):
    return np.minimum(G - 1, ((u + 1) * G - 1) // units)


def owner_def(u, units, G):
    starts = sk_start(np.arange(G + 1), units, G)
    return np.searchsorted(starts[:G], u, side="right") - 1


@pytest.mark.parametrize("tiles,kb", [(20, 128), (64, 32), (64, 112), (96, 64), (172, 64), (250, 128),
                                      (32, 64), (4096, 172), (1, 3), (7, 5)])
def test_owner_closed_form_matches_definition(tiles, kb):
    units = tiles * kb
    G = min(units, 148)
    assert units * G < 2 ** 31          # the kernels' 32-bit arithmetic
    u = np.arange(units)
    assert np.array_equal(owner_closed(u, units, G), owner_def(u, units, G))
    # contributors of each tile: later ones begin inside the tile (their first segment)
    for t in range(tiles):
        c0, c1 = owner_closed(t * kb, units, G), owner_closed((t + 1) * kb - 1, units, G)
        for c in range(c0 + 1, c1 + 1):
            assert sk_start(c, units, G) > t * kb
        # one contributor <=> the whole tile is one CTA's range
        whole = sk_start(c0, units, G) <= t * kb and sk_start(c0 + 1, units, G) >= (t + 1) * kb
        assert (c0 == c1) == whole
