"""Golden vectors for hand-built .sif streams, produced by the REFERENCE (slicer-codec 0.1.0).

The encoder never emits these, but decode() must treat them exactly like the reference:
cross-plane overlap (legal: the two planes are summed in float64, codec.py:257-266),
within-plane overlap, non-increasing cols, col >= K (CorruptStreamError, codec.py:235-251),
and multi-row planes with empty rows.  Run in the build container (needs /root/reference):

    python tests/golden/make_structural_golden.py   # writes tests/golden/structural.npz
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from slicer.codec import CompressedIF, EncodedBlock, decode, deserialize, serialize  # noqa: E402
from slicer.errors import SlicerError  # noqa: E402


def blk(q, o, vmin, row_ptr, cols, codes):
    return EncodedBlock(q=q, o=float(np.float32(o)), v_min=float(np.float32(vmin)), v_max=0.0, degenerate=False,
                        row_ptr=np.asarray(row_ptr, np.uint32), cols=np.asarray(cols, np.uint32),
                        codes=np.asarray(codes, np.uint32))


def cif(rows, cols, plus, minus):
    return CompressedIF(rows=rows, cols=cols, s=0.5, lam=0.0, q_bit=8, delta=0.01, mode="abq",
                        m_plus=len(plus), m_minus=len(minus), q_vector=(), blocks_plus=tuple(plus),
                        blocks_minus=tuple(minus))


def _random_cif(rows, cols, mp, mm, dens, seed, break_at=None):
    """Random planes with cross-plane overlaps; break_at swaps two cols around that column
    of one minus row (non-increasing -> CorruptStreamError)."""
    rng = np.random.default_rng(seed)

    def plane(m, minus):
        out = []
        for bi in range(m):
            q = int(rng.integers(1, 17))
            rp, cs, codes = [0], [], []
            for r in range(rows):
                cc = np.sort(rng.choice(cols, size=int(rng.binomial(cols, dens / m)), replace=False))
                if minus and break_at is not None and bi == 0 and r == 1 and len(cc) > 2:
                    j = int(np.searchsorted(cc, break_at))
                    j = min(max(j, 1), len(cc) - 1)
                    cc[j - 1], cc[j] = cc[j], cc[j - 1]
                cs += [int(c) for c in cc]
                codes += [int(x) for x in rng.integers(0, 1 << q, size=len(cc))]
                rp.append(len(cs))
            out.append(blk(q, float(rng.uniform(0.01, 2)), float(rng.uniform(0, 3)), rp, cs, codes))
        return out

    # blocks of a plane must not overlap each other: carve one plane's columns per block
    def disjoint(m, minus):
        bl = plane(m, minus)
        seen = [set() for _ in range(rows)]
        fixed = []
        for b in bl:
            rp, cs, codes = [0], [], []
            for r in range(rows):
                for k in range(int(b.row_ptr[r]), int(b.row_ptr[r + 1])):
                    c = int(b.cols[k])
                    if c in seen[r] and not (break_at is not None and minus):
                        continue
                    seen[r].add(c)
                    cs.append(c)
                    codes.append(int(b.codes[k]))
                rp.append(len(cs))
            fixed.append(blk(b.q, b.o, b.v_min, rp, cs, codes))
        return fixed

    return cif(rows, cols, disjoint(mp, False), disjoint(mm, True))


CASES = {
    # plus and minus planes share (0,1) and (2,3): float64 sums, not an error
    "cross_plane_overlap": cif(3, 5, [blk(8, 0.0123, 0.5, [0, 2, 2, 3], [1, 4, 3], [200, 7, 255])],
                               [blk(5, 0.77, 0.25, [0, 1, 1, 2], [1, 3], [31, 3])]),
    # rows without entries, several blocks per plane, odd widths
    "multi_block_rows": cif(4, 37, [blk(3, 1.5, 2.0, [0, 0, 2, 2, 3], [0, 36, 5], [7, 1, 4]),
                                    blk(1, 0.5, 1.0, [0, 1, 1, 1, 1], [20], [1])],
                            [blk(12, 0.001, 0.01, [0, 0, 0, 1, 2], [9, 0], [4095, 17])]),
    "within_plane_overlap": cif(2, 4, [blk(8, 0.5, 1.0, [0, 1, 1], [2], [3]), blk(8, 0.5, 2.0, [0, 1, 1], [2], [1])],
                                [blk(8, 1.0, 0.0, [0, 0, 0], [], [])]),
    "cols_not_increasing": cif(2, 8, [blk(4, 0.25, 0.0, [0, 2, 2], [5, 3], [1, 2])], [blk(8, 1.0, 0.0, [0, 0, 0], [], [])]),
    "cols_equal": cif(1, 8, [blk(4, 0.25, 0.0, [0, 2], [4, 4], [1, 2])], [blk(8, 1.0, 0.0, [0, 0], [], [])]),
    "col_ge_K": cif(2, 6, [blk(4, 0.25, 0.0, [0, 1, 2], [2, 7], [1, 2])], [blk(8, 1.0, 0.0, [0, 0, 0], [], [])]),
    # plus value rounds to an infinite fp32 alone, but the float64 plane sum is finite
    "cross_plane_inf_cancel": cif(1, 6, [blk(8, 3.0e38, 0.0, [0, 2], [1, 4], [255, 1])],
                                  [blk(8, 3.0e38, 0.0, [0, 1], [1], [254])]),
    "plus_inf": cif(1, 6, [blk(8, 3.0e38, 0.0, [0, 1], [2], [255])], [blk(8, 1.0, 0.0, [0, 0], [], [])]),
    "minus_inf": cif(1, 6, [blk(8, 1.0, 0.0, [0, 0], [], [])], [blk(8, 3.0e38, 0.0, [0, 1], [2], [255])]),
    # rows wider than a decode work item (column segments) and many (block, row) pairs
    "wide_rows": _random_cif(3, 2500, 3, 2, 0.2, 11),
    "many_pairs": _random_cif(70, 7, 4, 3, 0.5, 12),
    "wide_rows_bad": _random_cif(3, 2500, 3, 2, 0.2, 13, break_at=1900),
}


def main():
    arrays = {}
    names = []
    for name, c in CASES.items():
        data = serialize(c)
        arrays[f"{name}_blob"] = np.frombuffer(data, np.uint8)
        try:
            y = decode(deserialize(data))
            arrays[f"{name}_dec"] = y.values.copy()
            arrays[f"{name}_err"] = np.frombuffer(b"", np.uint8)
        except SlicerError as e:
            arrays[f"{name}_err"] = np.frombuffer(type(e).__name__.encode(), np.uint8)
            arrays[f"{name}_msg"] = np.frombuffer(str(e).encode(), np.uint8)
        names.append(name)
        print(name, len(data), hashlib.sha256(data).hexdigest()[:16],
              arrays[f"{name}_err"].tobytes().decode() or "ok")
    arrays["names"] = np.array(names)
    np.savez(os.path.join(HERE, "structural.npz"), **arrays)


if __name__ == "__main__":
    main()
