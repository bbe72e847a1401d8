"""Known-answer fixtures restated from the reference test suite (tests/test_runtime.cpp,
tests/test_compiler.cpp, tests/test_spline.cpp). Shared by the oracle tests and the GPU
parity tests so both are held to the same answers."""
import numpy as np


def hand_artifact_arrays(bm: int, op: int) -> dict:
    """test_runtime.cpp:19-34: one edge, knots {0,1,2}, L=4, uint8 codes, scale 1, phi."""
    return dict(in_dim=1, out_dim=1, L=4, knots=np.array([0, 1, 2], np.float32),
                q=np.array([0, 10, 20, 30, 40, 50, 60, 70], np.uint8), scale=np.ones(2, np.float32),
                y_min=np.zeros(2, np.float32), value_repr=0, scheme=1, boundary_mode=bm, oob_policy=op)


# (x, expected value, expected was_oob) under closed + clip_x (test_runtime.cpp:127-143)
HAND_CLOSED_CLIPX = [(0.0, 0.0, False), (0.5, 15.0, False), (1.0, 40.0, False), (1.5, 55.0, False),
                     (2.0, 70.0, False), (2.5, 70.0, True), (1e9, 70.0, True), (-55.0, 0.0, True)]
# half_open + zero_spline (test_runtime.cpp:145-161)
HAND_HALFOPEN_ZS = [(2.0, 0.0, True), (1.9999, None, False)]
# closed + zero_spline
HAND_CLOSED_ZS = [(2.0, 70.0, False), (2.1, 0.0, True)]

# test_compiler.cpp:93-114
SYM_EXAMPLE = ([-2.54, 0.0, 1.27, 2.54], [-127, 0, 64, 127], 0.02)
ASYM_EXAMPLE = ([1.0, 2.275, 3.55], [0, 128, 255], 0.01, 1.0)

# test_spline.cpp:101-127 cardinal B-spline values on uniform knots
CARDINAL = [((0.0, 1.0, 2.0, 3.0), 2, 1.5, [0.0, 1 / 8, 6 / 8, 1 / 8, 0.0]),
            ((0.0, 1.0, 2.0, 3.0), 3, 1.0, [0.0, 1 / 6, 4 / 6, 1 / 6, 0.0, 0.0]),
            ((0.0, 1.0, 2.0), 1, 0.5, [0.5, 0.5, 0.0]),
            ((0.0, 1.0, 2.0), 0, 1.0, [0.0, 1.0])]
