"""CPU: the host-side dictionary builders against the reference's own outputs.

``build_dictionary`` (reference dictionary.py:109-142: rotation-major, then
length, then origin; atoms that lose a pixel to the border dropped; exact
duplicates removed; binary columns) must reproduce the atoms the reference
enumerated for the same specs (tests/golden/known.npz ``dict_*``, written by
tests/golden/make_golden.py from the reference itself), column for column.
"""

import math

import numpy as np

from conftest import golden
from paper_2603_08582_b200.dictionary import (
    DictionarySpec,
    build_dictionary,
    build_extended_dictionary,
)

SPECS = {"s16_l4_r0_90": ((4,), (0.0, math.pi / 2), 16),
         "s16_l4_r4": ((4,), tuple(k * math.pi / 4 for k in range(4)), 16),
         "s12_l3l5_r8": ((3, 5), tuple(k * math.pi / 8 for k in range(8)), 12)}


def test_build_dictionary_matches_reference_atoms():
    g = golden("known.npz")
    for name, (lengths, rots, side) in SPECS.items():
        ref = g[f"dict_{name}_atoms"].astype(np.float64)
        d = build_dictionary(DictionarySpec(lengths, rots, side))
        assert d.atoms.shape == ref.shape, name
        assert np.array_equal(d.atoms, ref), name


def test_reference_dictionary_counts():
    # the reference's known answers (reference tests/test_dictionary.py:54-63)
    d = build_dictionary(DictionarySpec((4,), (0.0, 0.5 * math.pi), 16))
    assert d.m_atoms == 416 and d.n_pixels == 256
    assert build_dictionary(DictionarySpec((2, 4, 6), (0.0,), 16)).m_atoms == 624


def test_extended_dictionary_sizes_and_norms():
    # BASELINE cfg0 / cfg1 / cfg4 dictionaries
    for side, length, rot, stride, m in ((32, 4, 4, 1, 5120), (64, 6, 8, 1, 36864),
                                         (16, 4, 4, 2, 512)):
        d = build_extended_dictionary(side, length, rot, stride)
        assert d.m_atoms == m
        norms = np.sqrt((d.ell_w ** 2).sum(axis=1))
        assert np.allclose(norms, 1.0, rtol=1e-15)
