"""Host-side logic of the config-5 HELR-style driver (no GPU needed)."""
from paper_2407_13055_b200.helr import HelrShape


def test_helr_shape_rotations():
    sh = HelrShape(n=1 << 16, features=256, cts=8)
    assert sh.samples_per_ct == 128
    assert sh.feature_rotations() == [1, 2, 4, 8, 16, 32, 64, 128]
    assert sh.sample_rotations() == [256 << k for k in range(7)]
    small = HelrShape(n=1024, features=16, cts=4)
    assert small.rotations() == [1, 2, 4, 8, -1, -2, -4, -8, 16, 32, 64, 128, 256]

