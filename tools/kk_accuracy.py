"""KK field accuracy of the GPU kernel vs the oracle (rel L2) on goldens."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np
from oracle import kkoracle as ko
from paper_2108_07001_b200 import rxdsp
from paper_2108_07001_b200.captures import load_capture
for name in ["c1_qpsk_b2b", "c4_qpsk_10000km_cspr4", "c3_64qam_1600km_rel-20", "c4_qpsk_10000km_cspr14"]:
    cap = load_capture(name)
    x = cap.adc_float()[: 1 << 17]
    ref, _, _ = ko.kk_reconstruct(x, 1024)
    out, _, _ = rxdsp.kk_reconstruct(rxdsp.RealSignal(x, 4e9), rxdsp.BlockPlan(1024, buffer_len=len(x)))
    print(name, "kk rel L2", np.linalg.norm(out.samples - ref) / np.linalg.norm(ref))
