"""Adam and the step learning-rate schedule ("Adam optimizer ...
beta1=0.9 and beta2=0.999 ... learning rate schedule that starts at 1e-2 and
decays by a factor of 0.8 every 500 steps").

R12: PyTorch torch.optim.Adam semantics (the paper trained in PyTorch,
P:L215): eps = 1e-8, dense update of every entry, no weight decay.
R13: lr at 0-based step s is lr0 * 0.8^floor(s/500).
"""
import math
import numpy as np


def lr_at(s, lr0=1e-2, decay=0.8, every=500):
    return lr0 * decay ** (s // every)


def adam_update(p, g, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """One in-place update at 1-based step t (PyTorch form):
    m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2;
    p <- p - (lr / (1 - b1^t)) * m / (sqrt(v) / sqrt(1 - b2^t) + eps)."""
    m *= beta1
    m += (1.0 - beta1) * g
    v *= beta2
    v += (1.0 - beta2) * g * g
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    denom = np.sqrt(v) / math.sqrt(bc2) + eps
    p -= (lr / bc1) * m / denom
