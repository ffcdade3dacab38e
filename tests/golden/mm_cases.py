# SPDX-License-Identifier: Apache-2.0
"""MatrixMarket inputs for the loader parity tests (tests/test_matrix_market.py).

Deterministic texts: the hand cases of the reference's test_matrix_market.cpp
restated, every error branch of load_matrix_market (matrix_market.cpp:61-166),
the stream-extraction corner cases of its number parsing, and larger seeded
matrices in symmetric and general form with shuffled entry order.
make_golden.py records the reference's result for each case by name.
"""
from __future__ import annotations

import numpy as np

SYM = "%%MatrixMarket matrix coordinate real symmetric\n"
GEN = "%%MatrixMarket matrix coordinate real general\n"


def _sym_lap2d(nx, rng, jitter=True):
    """Lower triangle of a 2D 5-point pattern with seeded values (17 significant digits)."""
    ent = []
    for j in range(nx):
        for i in range(nx):
            r = j * nx + i
            ent.append((r, r, 4.0 + (rng.random() if jitter else 0.0)))
            if i > 0:
                ent.append((r, r - 1, -1.0 - (rng.random() / 3 if jitter else 0.0)))
            if j > 0:
                ent.append((r, r - nx, -1.0 - (rng.random() / 7 if jitter else 0.0)))
    return nx * nx, ent


def _fmt(v):
    return repr(float(v))


def _text(header, n, lines, declared=None):
    body = "".join(lines)
    return f"{header}{n} {n} {len(lines) if declared is None else declared}\n{body}"


def cases():
    c = {}
    # --- the reference's own hand cases (test_matrix_market.cpp:25-85)
    c["sym_2x2"] = SYM + "2 2 3\n1 1 2.0\n2 1 -1.0\n2 2 2.0\n"
    c["general_full"] = GEN + "% a comment\n2 2 4\n1 1 2.0\n1 2 -1.0\n2 1 -1.0\n2 2 2.0\n"
    c["zero_based"] = SYM + "2 2 1\n0 0 1.0\n"
    c["general_asym"] = GEN + "2 2 4\n1 1 2.0\n1 2 -1.0\n2 1 -1.5\n2 2 2.0\n"
    c["count_short"] = SYM + "2 2 3\n1 1 2.0\n"
    c["rect"] = SYM + "2 3 1\n1 1 2.0\n"
    c["complex"] = "%%MatrixMarket matrix coordinate complex symmetric\n1 1 1\n1 1 1.0\n"
    c["not_mm"] = "not a matrix market file\n"
    # --- header / size-line branches
    c["empty"] = ""
    c["banner_only"] = SYM
    c["comments_only"] = SYM + "% nothing\n%\n"
    c["size_two_numbers"] = SYM + "2 2\n1 1 1.0\n"
    c["size_zero"] = SYM + "0 0 0\n"
    c["size_text"] = SYM + "two 2 1\n"
    c["pattern"] = "%%MatrixMarket matrix coordinate pattern symmetric\n1 1 1\n1 1\n"
    c["array"] = "%%MatrixMarket matrix array real general\n1 1\n1.0\n"
    c["hermitian"] = "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1.0\n"
    c["banner_case"] = "%%matrixmarket matrix coordinate real symmetric\n1 1 1\n1 1 1.0\n"
    c["header_case"] = "%%MatrixMarket MATRIX Coordinate REAL Symmetric\n1 1 1\n1 1 5.0\n"
    c["header_short"] = "%%MatrixMarket matrix coordinate\n1 1 1\n1 1 1.0\n"
    c["vector_object"] = "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1.0\n"
    # --- entry branches
    c["count_long"] = SYM + "2 2 1\n1 1 2.0\n2 2 2.0\n"
    c["upper_in_symmetric"] = SYM + "2 2 2\n1 1 2.0\n1 2 -1.0\n"
    c["index_high"] = SYM + "2 2 1\n3 1 1.0\n"
    c["index_negative"] = SYM + "2 2 1\n-1 1 1.0\n"
    c["dup_symmetric"] = SYM + "2 2 3\n1 1 2.0\n2 1 -1.0\n2 1 -1.0\n"
    c["dup_general"] = GEN + "2 2 5\n1 1 2.0\n1 2 -1.0\n2 1 -1.0\n2 1 -1.0\n2 2 2.0\n"
    c["general_unpaired_tiny"] = GEN + "2 2 3\n1 1 2.0\n2 1 1e-20\n2 2 2.0\n"
    c["general_unpaired"] = GEN + "2 2 3\n1 1 2.0\n2 1 -1.0\n2 2 2.0\n"
    c["general_upper_only_paired"] = GEN + "3 3 5\n1 1 2.0\n1 3 -0.5\n3 1 -0.5000000000000001\n2 2 2.0\n3 3 2.0\n"
    c["crlf"] = SYM.replace("\n", "\r\n") + "2 2 3\r\n1 1 2.0\r\n2 1 -1.0\r\n2 2 2.0\r\n"
    c["blank_lines"] = SYM + "\n2 2 3\n\n1 1 2.0\n\n2 1 -1.0\n2 2 2.0\n\n"
    c["space_line"] = SYM + "2 2 3\n1 1 2.0\n \n2 1 -1.0\n2 2 2.0\n"
    c["cr_only_line"] = SYM + "2 2 3\n1 1 2.0\n\r\n2 1 -1.0\n2 2 2.0\n"
    c["indented_comment"] = SYM + "2 2 2\n1 1 2.0\n  % not a comment\n2 2 2.0\n"
    c["tabs_and_trailing"] = SYM + "2\t2\t3 extra\n1\t1\t2.0 trailing words\n2 1 -1.0 9 9\n2 2 2.0\n"
    c["no_final_newline"] = SYM + "2 2 3\n1 1 2.0\n2 1 -1.0\n2 2 2.0"
    c["comments_between"] = SYM + "% head\n2 2 3\n% mid\n1 1 2.0\n%\n2 1 -1.0\n% x\n2 2 2.0\n%end"
    # --- number extraction corner cases (std::istream >> long long / double)
    nums = {"plus_point": "+.5", "trailing_point": "1.", "neg_zero": "-0", "tiny": "1e-400",
            "denormal": "4.9e-324", "hexfloat": "0x1p3", "two_points": "1.5.5", "comma": "1,5",
            "exp_upper": "2.5E+2", "lead_zeros": "0003.2500", "huge": "1e400", "inf": "inf",
            "nan": "nan", "dot": ".", "bare_exp": "1e", "exp_sign_only": "1e+", "sign_only": "-",
            "long_mantissa": "3.14159265358979323846264338327950288419716939937510",
            "max_double": "1.7976931348623157e308", "int_value": "7"}
    for k, v in nums.items():
        c[f"num_{k}"] = SYM + f"1 1 1\n1 1 {v}\n"
    c["idx_float"] = SYM + "1 1 1\n1.0 1 2.0\n"
    c["idx_plus"] = SYM + "2 2 1\n+2 +1 2.0\n"
    c["idx_lead_zero"] = SYM + "2 2 1\n02 01 2.0\n"
    c["idx_overflow"] = SYM + "2 2 1\n99999999999999999999 1 2.0\n"
    c["idx_hex"] = SYM + "2 2 1\n0x2 1 2.0\n"
    c["value_missing"] = SYM + "2 2 1\n2 1\n"
    # --- seeded larger matrices
    rng = np.random.default_rng(2008_01440)
    n, ent = _sym_lap2d(30, rng)
    order = rng.permutation(len(ent))
    c["lap2d30_sym_shuffled"] = _text(SYM, n, [f"{ent[k][0] + 1} {ent[k][1] + 1} {_fmt(ent[k][2])}\n" for k in order])
    full = []
    for (i, j, v) in ent:
        full.append((i, j, v))
        if i != j:
            full.append((j, i, v))
    order = rng.permutation(len(full))
    c["lap2d30_general_shuffled"] = _text(GEN, n, [f"{full[k][0] + 1} {full[k][1] + 1} {_fmt(full[k][2])}\n" for k in order])
    # general with a tolerated mismatch: the lower value must win
    g2 = []
    for (i, j, v) in ent:
        g2.append((i, j, v))
        if i != j:
            g2.append((j, i, v * (1 + 1e-14)))
    order = rng.permutation(len(g2))
    c["lap2d30_general_near"] = _text(GEN, n, [f"{g2[k][0] + 1} {g2[k][1] + 1} {_fmt(g2[k][2])}\n" for k in order])
    # many threads' worth of lines (the loader splits bodies > 1 MiB into chunks)
    n, ent = _sym_lap2d(160, rng)
    order = rng.permutation(len(ent))
    c["lap2d160_sym_big"] = _text(SYM, n, [f"{ent[k][0] + 1} {ent[k][1] + 1} {_fmt(ent[k][2])}\n" for k in order])
    # ... with an error deep inside (the first failing line must be reported)
    lines = [f"{ent[k][0] + 1} {ent[k][1] + 1} {_fmt(ent[k][2])}\n" for k in order]
    lines[len(lines) * 3 // 4] = "1 2 5.0\n"         # upper entry (later line)
    lines[len(lines) // 2] = "7 7 bogus\n"           # malformed (earlier line: reported)
    c["lap2d160_sym_big_error"] = _text(SYM, n, lines)
    return {k: v.encode() for k, v in c.items()}
