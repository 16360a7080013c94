"""Small end-to-end receive for compute-sanitizer (memcheck / racecheck /
synccheck): the c4 golden capture through RxPipeline (K1, carrier, K2, sync,
DDLMS solver incl. training, scans, list passes) plus the packed-bit e2e path
(async DDLMS worker) and the capture generator."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_07001_b200 import rxdsp  # noqa: E402
from paper_2108_07001_b200.captures import load_capture  # noqa: E402
from paper_2108_07001_b200.harness import receive_host_stream  # noqa: E402

cap = load_capture("c4_qpsk_10000km_cspr10")
cfg = cap.pipeline_config(ddlms_frame_symbols=1 << 15)
pipe = rxdsp.RxPipeline(cfg, reference_symbols=cap.symbols())
pipe.feed(cap.adc)
dec, soft = pipe.finish()
print("decisions", len(dec))
_, bits, n = receive_host_stream(cfg, torch.from_numpy(cap.adc_h).pin_memory(), cap.half_lsb, cap.symbols(),
                                 chunk_samples=1 << 16)
torch.cuda.synchronize()
print("stream decisions", n)

# round-2 additions: frame sync correlation, metrics kernels, any-length FFT,
# split-step span, packed 12-bit input, general tone
from types import SimpleNamespace  # noqa: E402

from paper_2108_07001_b200 import channel  # noqa: E402
from paper_2108_07001_b200.harness import measure_point_device  # noqa: E402
from paper_2108_07001_b200.sigcore import ComplexSignal, AdcPacked12, pack12  # noqa: E402

lab, soft_d, _ = (lambda p: (p.feed(cap.adc), p.feed(np.zeros(0), flush=True), p.drain_device())[-1])(
    rxdsp.RxPipeline(cfg, reference_symbols=cap.symbols()))
c = cap.meta["config"]
cfgx = SimpleNamespace(tx=SimpleNamespace(constellation_order=4, baud_hz=c["tx"]["baud_hz"]),
                       rx=SimpleNamespace(startup_symbols=c["rx"]["startup_symbols"]),
                       metrics=SimpleNamespace(head_guard_symbols=2048, tail_guard_symbols=4096,
                                               windowed_q_window_s=20e-6))
bits_ref = np.unpackbits(cap.arrays["bits_packed"])[: cap.meta["n_bits"]]
print("point", measure_point_device(lab, soft_d, bits_ref, cap.symbols(), cfgx)["n_errors"])
x = np.random.default_rng(1).standard_normal(5000) + 0j
print("fft", float(np.abs(channel.fft(x) - np.fft.fft(x)).max()))


class _Span:
    length_km, loss_db_per_km, dispersion_ps_nm_km, gamma_per_w_km = 50.0, 0.2, 17.0, 1.3


print("ssfm", len(channel.ssfm_span(ComplexSignal(x, 16e9), _Span(), 10.0)))
p12 = rxdsp.RxPipeline(cfg, reference_symbols=cap.symbols())
p12.feed(AdcPacked12(torch.from_numpy(pack12(cap.adc_h)).cuda(), cap.half_lsb, len(cap.adc_h)))
print("packed12", len(p12.finish()[0]))
import dataclasses  # noqa: E402
pt = rxdsp.RxPipeline(dataclasses.replace(cfg, tone_freq_hz=0.516e9 + 2.5), reference_symbols=cap.symbols())
pt.feed(cap.adc)
print("general tone", len(pt.finish()[0]))
torch.cuda.synchronize()
