"""SPEC acceptance criterion 4, counters only: at n = 2^15 slots
the BSGS method's rotations are < 10 % of the packed-row method's for the
Llama preset (4096 x 14336), and the row/BSGS gap widens monotonically across
the GPT-2 -> Phi-3 -> Llama presets.  Counts come from
helix::predicted_rotations (libhelix_b200.so, host only), which the GPU
acceptance test pins to the traced counts of real matvecs
(tests/test_gpu_acceptance.py)."""
import pytest

PRESETS = [("gpt2", 768, 3072), ("phi3", 3072, 8192), ("llama", 4096, 14336)]  # d_model x d_ffn


def test_row_vs_bsgs_rotation_ratio():
    from paper_2512_11135_b200.helix import BSGS, DIAG, ROW, predicted_rotations

    n = 1 << 15
    ratios = []
    for name, rows, cols in PRESETS:
        row = predicted_rotations(ROW, rows, cols, n)
        bsgs = predicted_rotations(BSGS, rows, cols, n)
        diag = predicted_rotations(DIAG, rows, cols, n)
        assert bsgs < row and bsgs < diag
        ratios.append(bsgs / row)
    assert ratios[-1] < 0.10
    assert ratios[0] > ratios[1] > ratios[2]  # BSGS share shrinks as the models grow


def test_predicted_rotation_closed_forms():
    from paper_2512_11135_b200.helix import BSGS, DIAG, ROW, predicted_rotations

    n = 1 << 12
    assert predicted_rotations(BSGS, 64, 64, n) == 14  # n1 = n2 = 8
    assert predicted_rotations(DIAG, 64, 64, n) == 63
    assert predicted_rotations(ROW, 64, 64, n) == 6 + 63  # one group: log2(64) + 63 shifts
    assert predicted_rotations(BSGS, 512, 256, n) == 15 + 2 * 15  # 2 row blocks share the baby steps
    with pytest.raises(Exception):
        predicted_rotations(BSGS, 4, 8192, n)  # wider than the slot count


def test_criterion_8_gelu_fit():
    """SPEC criterion 8 (cleartext part): a degree-127 Chebyshev fit of GeLU on
    [-8, 8] is within 1e-2 of exact GeLU on a 10^4-point grid (the coefficients
    polyeval takes for the paper's GeLU(degree=127))."""
    import numpy as np
    from scipy.special import erf

    gelu = lambda t: 0.5 * t * (1 + erf(t / np.sqrt(2)))  # noqa: E731
    fit = np.polynomial.chebyshev.Chebyshev.interpolate(gelu, 127, domain=[-8, 8])
    grid = np.linspace(-8, 8, 10_000)
    assert np.abs(fit(grid) - gelu(grid)).max() < 1e-2
