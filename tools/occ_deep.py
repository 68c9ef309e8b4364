"""Max co-resident clusters of the deep kernel per cluster size (cudaOccupancyMaxActiveClusters).

    PYTHONPATH=. python tools/occ_deep.py
"""
import ctypes, torch
from paper_2304_09590_b200 import load
L = load(); torch.zeros(1).cuda()
for C in (4, 5, 6, 7, 8, 10, 12, 16):
    print("deep C", C, "max active clusters", L.pnn_debug_deep_max_clusters(C))
