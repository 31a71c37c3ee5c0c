"""Probe how tcgen05.mma.kind::tf32 converts raw fp32 operands (truncate vs round).
FS_SYRK_DBG=64 makes the converters pass the raw fp32 value as 'hi' and zero 'lo', so the
Gram entry is tf32(x)^2 as the tensor core sees it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2310_17556_b200 as fsb
x = np.float32(1.0 + 0.75 * 2.0 ** -10)     # between tf32 neighbours 1 and 1 + 2^-10
S = np.zeros((1, 32), np.float32); S[0, 0] = x
W = fsb.gram(fsb.ScoreMatrix(S), 1e-30, precision="tf32x3")[0, 0]
print("x=%r  W=%r  trunc^2=%r  round^2=%r  exact=%r" % (float(x), W, 1.0, (1 + 2.0 ** -10) ** 2, float(x) ** 2))
y = np.float32(1.0 + 0.25 * 2.0 ** -10)
S[0, 0] = y
W = fsb.gram(fsb.ScoreMatrix(S), 1e-30, precision="tf32x3")[0, 0]
print("y=%r  W=%r" % (float(y), W))
