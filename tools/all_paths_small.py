"""Tiny runs of every training path (resident, cluster, reference, fp32 and bf16 mini-batch) with
merge, predict and evaluate: a quick all-kernels check (tools only)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from datagen import make_rows
from paper_2304_09590_b200 import PNN, PNN_BF16

def run(layers, act, K, n, kernel="auto", batch=1, prec=0, epochs=1):
    X, y = make_rows(0, n, "train", 0)
    net = PNN(layers, act, "he", K, 0.01, seed=0)
    net.set_kernel(kernel)
    if batch > 1:
        net.set_minibatch(batch, prec)
    xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    for _ in range(epochs):
        net.train_epoch(xd, yd)
    net.merge()
    lab = net.predict(xd[:37])
    acc = net.evaluate(xd[:37], yd[:37])
    torch.cuda.synchronize()
    net.close()
    print(layers, kernel, batch, prec, "ok", acc[0])

run([784, 128, 10], ["relu", "softmax"], 4, 4 * 9 + 3, "resident")
run([784, 100, 10], ["sigmoid", "sigmoid"], 2, 2 * 7 + 1, "resident")
run([784, 16, 10], ["tanh", "softmax"], 2, 2 * 5, "resident")
run([784, 300, 100, 10], ["tanh", "tanh", "softmax"], 2, 2 * 6 + 1, "cluster")
run([784, 64, 10], ["relu", "softmax"], 3, 3 * 20 + 2, "reference")
run([784, 256, 10], ["relu", "softmax"], 2, 2 * 60 + 7, "auto", batch=50)
run([784, 1024, 1024, 10], ["relu", "relu", "softmax"], 2, 2 * 70, "auto", batch=64, prec=PNN_BF16)
