import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import kkoracle as ko
from paper_2108_07001_b200 import rxdsp
from paper_2108_07001_b200.captures import load_capture
from paper_2108_07001_b200.constellation import make_constellation
cap = load_capture("c1_qpsk_b2b")
x = cap.adc_float().copy(); x[150000:150600] *= 100.0
ref, d_ref, s_ref = ko.receive(x, ko.OracleConfig(taps=cap.taps), cap.symbols(), 1 << 22)
P = make_constellation(4).points
ir = np.argmin(np.abs(d_ref[:,None]-P[None,:]),1)
for rep in range(3):
    for graph in ("1", "0"):
        os.environ["KK_DDLMS_GRAPH"] = graph
        import importlib; rxdsp._DDLMS_GRAPH = graph != "0"
        cfg = cap.pipeline_config()
        pipe = rxdsp.RxPipeline(cfg, reference_symbols=cap.symbols())
        pipe.feed(x)
        dec, soft = pipe.finish()
        idx = np.argmin(np.abs(dec[:,None]-P[None,:]),1)
        bad = np.nonzero(idx != ir)[0]
        st = pipe.ddlms_stats
        print(rep, graph, st[0]["mode"], st[0]["iterations"], st[0]["per_iter"][:6], "agree", np.mean(idx==ir), "first bad", bad[:3], "n", len(bad))
        if len(bad):
            k = bad[0]
            print("   soft gpu", soft[k-2:k+3]); print("   soft ref", s_ref[k-2:k+3])
