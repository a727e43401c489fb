"""Generate the fixture-format goldens with the REFERENCE's own writers.

Run in the build container (where /root/reference exists):
    python tests/golden/make_fixture_golden.py
Writes tests/golden/ref_matrix_fixture.txt (matstore.write_fixture, matstore.py:301-307),
tests/golden/ref_ocp_fixture.txt (apps.write_ocp_fixture, apps.py:323-331).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import import_reference  # noqa: E402

pb = import_reference()
from panelblas import apps, matstore  # noqa: E402


def main():
    rng = np.random.default_rng(20261022)
    a = rng.standard_normal((5, 3)) * np.array([1e-300, 1.0, 3e7])  # tiny / normal / large values
    a[0, 0] = -0.0
    cm = matstore.allocate_col_matrix(5, 3)
    for i in range(5):
        for j in range(3):
            cm.set(i, j, float(a[i, j]))
    matstore.write_fixture(os.path.join(HERE, "ref_matrix_fixture.txt"), cm)
    nx, nu, N = 2, 1, 2
    stages = []
    for _ in range(N):
        A, B = rng.standard_normal((nx, nx)), rng.standard_normal((nx, nu))
        Q, R, S = np.eye(nx) * 0.5, np.eye(nu) * 2.0, rng.standard_normal((nu, nx)) * 0.1
        stages.append(apps.RiccatiStage(A, B, Q, R, S))
    P = np.eye(nx) * 3.0
    apps.write_ocp_fixture(os.path.join(HERE, "ref_ocp_fixture.txt"),
                           apps.OcpData(apps.OcpDims(nx, nu, N), stages, P))
    print("wrote fixture goldens")


if __name__ == "__main__":
    main()
