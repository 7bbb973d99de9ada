"""Small MLP with ReLU hidden layers and a linear output layer (P:L157-158
"a small multilayer perceptron (MLP) network ... ReLU ... in the hidden
layers"; "4 hidden layers with 64 neurons each ... The output layer
does not use an activation function").

H hidden layers of width W => H+1 weight matrices: in->W, (H-1) x W->W, W->D
(R16).  Biases on by default (R15).  Float64.
"""
import numpy as np


def forward(weights, biases, feat):
    """weights[k]: (out_k, in_k); biases[k]: (out_k,) or None.
    z_k = h_{k-1} W_k^T + b_k; h_k = max(z_k, 0) for hidden k; y = z_last.
    Returns (y, zs, hs) where hs[0] = feat and zs are pre-activations."""
    h = np.asarray(feat, dtype=np.float64)
    hs, zs = [h], []
    for k, W in enumerate(weights):
        z = h @ W.T
        if biases[k] is not None:
            z = z + biases[k]
        zs.append(z)
        if k < len(weights) - 1:
            h = np.maximum(z, 0.0)
            hs.append(h)
        else:
            h = z
    return h, zs, hs


def backward(weights, biases, zs, hs, dy):
    """Reverse-mode differentiation of forward():
    dz_last = dy; dW_k = dz_k^T h_{k-1}; db_k = sum_i dz_k; dh_{k-1} = dz_k W_k;
    dz_{k-1} = dh_{k-1} * 1[z_{k-1} > 0] (ReLU'(0) = 0, R11).
    Returns (dW list, db list, dfeat)."""
    K = len(weights)
    dW = [None] * K
    db = [None] * K
    dz = np.asarray(dy, dtype=np.float64)
    for k in range(K - 1, -1, -1):
        dW[k] = dz.T @ hs[k]
        db[k] = dz.sum(axis=0) if biases[k] is not None else None
        dh = dz @ weights[k]
        if k > 0:
            dz = dh * (zs[k - 1] > 0.0)
        else:
            dfeat = dh
    return dW, db, dfeat
