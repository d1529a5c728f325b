"""Write Matrix Market fixtures with the UNMODIFIED reference (run here, not on
the GPU box): tests/golden/ref_block.mtx from a small block with edge values,
and tests/golden/ref_gen.mtx, the reference CLI's `gen -m 40 -n 3
--log10-cond 2.5 --seed 9` output.  The CPU/GPU tests check that this package
writes the same bytes and reads the same values.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mtx.py
"""

import os

import numpy as np
from cholqr.cli import main
from cholqr.varray import DenseVectorArray, save_matrix_market

HERE = os.path.dirname(os.path.abspath(__file__))

rng = np.random.default_rng(31)
block = rng.standard_normal((7, 3))
block[0, 0] = 1.0 / 3.0
block[1, 1] = -0.0
block[2, 2] = 1e-300
block[3, 0] = 123456789.125
block[4, 1] = 5e-324
block[5, 2] = -2.5e17
save_matrix_market(DenseVectorArray.from_numpy(block), os.path.join(HERE, "ref_block.mtx"))
assert main(["gen", "-m", "40", "-n", "3", "--log10-cond", "2.5", "--seed", "9", "-o",
             os.path.join(HERE, "ref_gen.mtx")]) == 0
