# Diagnostic (kept for reference): AUTO / SEGMENT / THROUGHPUT trackers on the same
# recordings give the same per-channel epoch counts; compare records with
# Tracker.records (records_raw also returns the unused, uninitialised ring slots).
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1907_00463_b200 import abi, simsource as ss
from paper_1907_00463_b200.tracking import Tracker, Context, init_channel_from_acquisition
ctx = Context(0)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
fs, ms = 65.472e6, 5
nrec = (2 * nsm + 11) // 12
rng = np.random.default_rng(5)
raws, inits, cstream = [], [], []
for r in range(nrec):
    prns = rng.choice(np.arange(1, 33), 12, replace=False)
    svs = [ss.Sv(prn=int(p), cn0_dbhz=45.0, doppler_hz=rng.uniform(-4000, 4000), delay_chips=rng.uniform(0, 1023)) for p in prns]
    for sv in svs:
        b, d = ss.truth_channel_start(sv, fs)
        inits.append(init_channel_from_acquisition(sv.prn, d, 0, b, 0, fs))
    cstream += [r] * 12
    raws.append(svs)
print("offsets", [int(c.sample_offset_next_epoch) for c in inits[:12]])
dev = ss.synth_gpu(ctx, ms, fs, raws, seed=9)
taps = abi.Taps.make([-0.75 + 0.25 * k for k in range(7)], early=4, prompt=3, late=2)
res = {}
for mode in (abi.CTA_AUTO, abi.CTA_SEGMENT, abi.CTA_THROUGHPUT):
    trk = Tracker(ctx, abi.FMT_INT16_IQ, fs, 0.0, inits, chan_stream=cstream, n_streams=nrec, taps=taps,
                  ring_samples=(ms + 4) * 65472, max_records=ms, cta_mode=mode)
    if mode != abi.CTA_THROUGHPUT:
        trk.attach_device(dev.data_ptr(), dev.shape[1] // 4, dev.shape[1])
    else:
        trk.push_device_strided(dev.data_ptr(), dev.shape[1], dev.shape[1])
    trk.run(); trk.sync()
    res[mode] = (trk.epoch_counts(), trk.records_raw())
    print(mode, np.bincount(res[mode][0]))
for mode in (abi.CTA_AUTO, abi.CTA_SEGMENT):
    d = np.nonzero(res[mode][0] != res[abi.CTA_THROUGHPUT][0])[0]
    print("mode", mode, "count diffs vs throughput:", len(d), d[:10], res[mode][0][d[:5]], res[abi.CTA_THROUGHPUT][0][d[:5]])
