"""NEXT-1: the boundary loss of Eq. 2 improves continuity across
the shared face, on a synthetic 2x1x1 split."""
import pytest

from studies import lambda_sweep

pytestmark = pytest.mark.gpu


def test_boundary_loss_reduces_face_mismatch():
    res = {r["lambda"]: r for r in lambda_sweep.run(steps=600, lambdas=(0.0, 0.5))}
    print(res)
    assert res[0.5]["slice_mismatch_rms"] < res[0.0]["slice_mismatch_rms"]
    assert res[0.5]["slice_psnr_mean_db"] > res[0.0]["slice_psnr_mean_db"]
