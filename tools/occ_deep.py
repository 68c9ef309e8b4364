"""Max co-resident clusters of the deep kernel per cluster size (cudaOccupancyMaxActiveClusters).

    PYTHONPATH=. python tools/occ_deep.py
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_09590_b200 import load
L = load(); torch.zeros(1).cuda()
for C in (4, 8):
    print("deep C", C, "max active clusters", L.pnn_debug_deep_max_clusters(C))
