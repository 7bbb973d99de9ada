"""Pins of oracle/render.py (NEXT-3) against closed forms."""
import math

import numpy as np

from oracle import render as R

CAM = dict(eye=(8.0, 8.0, -30.0), look=(8.0, 8.0, 8.0), up=(0.0, 1.0, 0.0), fovy=30.0, width=9, height=7)
LO, HI = (0.0, 0.0, 0.0), (16.0, 16.0, 16.0)


def tf(points, rgba, base_step=1.0):
    return dict(points=points, rgba=rgba, vmin=0.0, vmax=1.0, base_step=base_step)


def test_transparent_tf_gives_black_clear():
    frag = R.render_brick(lambda p: 0.5, CAM, LO, HI, 0.5, tf([0.0, 1.0], [[1, 0, 0, 0], [0, 1, 0, 0]]))
    assert np.all(frag[:, :4] == 0)


def test_single_opaque_sample_saturates():
    # a_tf = 1 -> that sample's colour, alpha 1
    f = tf([0.0, 1.0], [[0.2, 0.4, 0.6, 1.0], [0.2, 0.4, 0.6, 1.0]])
    C, A = R.ray_segment(lambda p: 0.3, np.zeros(3), np.array([0, 0, 1.0]), 0.0, 10.0, 1.0, f)
    assert A == 1.0 and np.allclose(C, [0.2, 0.4, 0.6], atol=1e-15)


def test_opacity_correction_closed_form():
    """Constant field, a_tf = a0, n samples of step s: 1 - A = (1 - a0)^(n s / b),
    C = c A (emission-absorption with step correction)."""
    a0, s, b = 0.1, 0.25, 0.5
    f = tf([0.0, 1.0], [[1.0, 0.5, 0.0, a0], [1.0, 0.5, 0.0, a0]], base_step=b)
    C, A = R.ray_segment(lambda p: 0.7, np.zeros(3), np.array([0, 0, 1.0]), 0.0, 3.0, s, f, stop_alpha=2.0)
    n = 12                                           # t_k = 0.125, 0.375, ..., 2.875
    assert abs((1 - A) - (1 - a0) ** (n * s / b)) < 1e-14
    assert np.allclose(C, np.array([1.0, 0.5, 0.0]) * A, atol=1e-14)


def test_sample_positions_are_global():
    # t_k = (k + 0.5) step from the eye, whatever the brick
    seen = []
    R.ray_segment(lambda p: seen.append(p[2]) or 0.0, np.zeros(3), np.array([0, 0, 1.0]), 1.1, 2.6, 0.5,
                  tf([0.0, 1.0], [[0, 0, 0, 0]] * 2))
    assert seen == [1.25, 1.75, 2.25]


def test_split_ray_composites_to_the_unsplit_result():
    """S:L514 compositing associativity: splitting the interval at an interior
    plane and compositing the two fragments equals the unsplit ray (1e-12)."""
    field = lambda p: 0.5 + 0.5 * math.sin(0.3 * p[0] + 0.2 * p[1] + 0.25 * p[2])
    f = tf([0.0, 0.3, 0.7, 1.0], [[0, 0, 1, 0.0], [0, 1, 0, 0.05], [1, 1, 0, 0.2], [1, 0, 0, 0.6]])
    whole = R.render_brick(field, CAM, LO, HI, 0.37, f, stop_alpha=2.0)
    front = R.render_brick(field, CAM, (0.0, 0.0, 0.0), (16.0, 16.0, 6.3), 0.37, f, stop_alpha=2.0)
    back = R.render_brick(field, CAM, (0.0, 0.0, 6.3), (16.0, 16.0, 16.0), 0.37, f, stop_alpha=2.0)
    img1 = R.composite([whole])
    img2 = R.composite([back, front])           # arrival order does not matter (depth sort)
    assert np.max(np.abs(img1 - img2)) < 1e-12
    assert np.max(img1[:, 3]) > 0.5


def test_step_convergence():
    """halving the step changes pixel values by < 1e-2 on a smooth field."""
    field = lambda p: 0.5 + 0.4 * math.sin(0.2 * p[0]) * math.cos(0.15 * p[2])
    f = tf([0.0, 1.0], [[0, 0, 1, 0.02], [1, 0, 0, 0.1]])
    a = R.composite([R.render_brick(field, CAM, LO, HI, 0.2, f)])
    b = R.composite([R.render_brick(field, CAM, LO, HI, 0.1, f)])
    assert np.max(np.abs(a - b)) < 1e-2


def test_background_and_misses():
    cam = dict(CAM, look=(8.0, 60.0, 8.0))           # looking away: every ray misses
    frag = R.render_brick(lambda p: 0.5, cam, LO, HI, 0.5, tf([0.0, 1.0], [[1, 1, 1, 1]] * 2))
    assert np.all(np.isinf(frag[:, 4]))
    img = R.composite([frag], background=(0.1, 0.2, 0.3))
    assert np.allclose(img, [0.1, 0.2, 0.3, 0.0])


def test_center_ray_points_at_the_look_point():
    d = R.camera_rays((0, 0, 0), (0, 0, 5), (0, 1, 0), 40.0, 3, 3)
    right = np.cross([0, 0, 1], [0, 1, 0])                  # r = f x up
    assert np.allclose(d[4], [0, 0, 1]) and d[0][1] > 0 and d[0] @ right < 0   # top-left: up and to the left
    # the corner ray's angle to the axis: tan = sqrt(a^2 + b^2), a = (2/3)(1/3... ) tan(20 deg)
    th = math.tan(math.radians(20.0))
    a, b = (2 * 0.5 / 3 - 1) * th, (1 - 2 * 0.5 / 3) * th
    assert abs(math.atan2(math.hypot(d[0][0], d[0][1]), d[0][2]) - math.atan(math.hypot(a, b))) < 1e-12


def test_batched_field_equals_per_sample_field():
    field = lambda p: 0.5 + 0.5 * math.sin(0.3 * p[0] - 0.2 * p[2])
    f = tf([0.0, 0.5, 1.0], [[0, 0, 1, 0.0], [0, 1, 0, 0.3], [1, 0, 0, 0.9]])
    a = R.render_brick(field, CAM, LO, HI, 0.5, f)
    b = R.render_brick(None, CAM, LO, HI, 0.5, f, batch_field=lambda P: np.array([field(p) for p in P]))
    assert np.array_equal(a, b)
