"""bench.py's roofline byte rule (host logic, no GPU): kept rows read every
tested mask, a row removed at pass t reads one witness mask (Lemma 1);
full-check bytes = SURVEY §8(d)'s Σ_t Σ_x |D_{t-1}(x)| · |changed neighbours| · d/8.
Checked against a hand-counted 3-variable chain."""
import numpy as np

import bench


def test_pass_bytes_chain():
    # complete graph on 3 variables, d = 8 (1 byte per mask); D_in: x0 {0,1}, x1 {0,1,2}, x2 {0}
    d = 8
    live0 = np.zeros((3, d), dtype=bool)
    live0[0, :2] = live0[1, :3] = live0[2, 0] = True
    remd = np.zeros((3, d), dtype=np.int32)
    remd[1, 2] = 1          # pass 1 removes (x1, 2)
    remd[0, 1] = 2          # pass 2 removes (x0, 1)

    def nbr_count(chg):
        return chg.sum() - chg.astype(np.int64)

    lpp, alg, full = bench.pass_bytes(live0, remd, 3, nbr_count, np.ones(3, dtype=bool), d)
    # pass 1: every column tested, 2 neighbours each; 6 live rows; (x1,2) removed
    # pass 2: changed = {x1}: x0 and x2 test it (1 each), x1 tests none; 5 live rows; (x0,1) removed
    # pass 3: changed = {x0}: x1 (2 rows) and x2 (1 row) test it; nothing removed
    assert lpp == [6, 5, 4]
    assert full == 6 * 2 + (2 * 1 + 2 * 0 + 1 * 1) + (1 * 0 + 2 * 1 + 1 * 1)
    assert alg == (5 * 2 + 1) + (1 * 1 + 1 + 1 * 1) + 3
