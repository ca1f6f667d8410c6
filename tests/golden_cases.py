"""Fixture case lists shared by tests/golden/make_golden.py and the tests."""

DEEPR_CASES = [
    # name, num_pre, num_post, density, seed, exclude_diag, headroom, cycles
    ("small16", 16, 16, 0.2, 3, False, 2.0, 4),
    ("adv32", 32, 32, 0.15, 12, False, 2.0, 4),
    ("diag12", 12, 12, 0.3, 13, True, 2.0, 4),
    ("full6x8", 6, 8, 0.5, 14, False, 1.0, 3),
    ("wide64x700", 64, 700, 0.1, 21, False, 2.0, 3),
    ("rec256", 256, 256, 0.1, 22, True, 2.0, 2),
    ("tight40", 40, 24, 0.6, 23, False, 1.05, 4),
]
