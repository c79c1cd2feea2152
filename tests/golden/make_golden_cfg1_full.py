"""Oracle history of the full BASELINE cfg1 run (160x80, 50 iterations, explicit
level-set scheme, reinit every 5) -- the parity fixture for the north star's
"J/C history within 1e-4 over the config's iteration count" at the config's own
size.  CPU only (~3 min):

    python tests/golden/make_golden_cfg1_full.py

Writes tests/golden/oracle_cfg1_full.npz.  The oracle itself is pinned to the
reference's own run() history (tests/test_oracle.py).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import cases as ocases, driver as odriver  # noqa: E402
from paper_2601_05709_b200 import configs  # noqa: E402


def main():
    c = configs.case("cfg1")
    grid, om, ovel, ophi, oparams, h = ocases.build(c)
    _, hist = odriver.run(om, ovel, ophi, oparams, h)
    keys = ("cost", "lagrangian", "form_value", "steps", "nsub_transport", "nsub_reinit")
    out = {k: np.array([r[k] for r in hist]) for k in keys}
    out["constraint"] = np.array([r["constraint"][0] for r in hist])
    np.savez_compressed(os.path.join(HERE, "oracle_cfg1_full.npz"), **out)
    print(len(hist), out["cost"][[0, -1]])


if __name__ == "__main__":
    main()
