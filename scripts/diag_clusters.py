"""Resident clusters of the cluster-sweep kernel by cluster size (cudaOccupancyMaxActiveClusters)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2303_08881_b200 import device as D

torch.zeros(1, device="cuda")
print({c: D.query("ddilu_csweep_active_clusters", c, 400) for c in range(1, 17)}, flush=True)
