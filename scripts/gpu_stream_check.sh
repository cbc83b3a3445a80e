#!/bin/bash
# Streamed path checks: parity of the early-stop frame queue and the TMA kernel, then speeds.
python -m pytest tests -m gpu -q -k "tma_staging or streamed_equals_resident or stream_frame_queue or c4_long" 2>&1 | tail -4
python scripts/c4_es_speed.py 65536 1.1 2>&1 | tail -6
python - <<'PY'
import time, torch, sys
sys.path.insert(0, ".")
import paper_1202_1060_b200 as P
g = P.configs.c4_code(); s = P.configs.c4_schedules(g)["ndgsbp"]
for ebn0 in (1.1, 1.3):
    s2 = P.sigma2_from_ebn0(ebn0, g.rate)
    P.simulate(g, s, s2, 1, 0, 8192, 30, early_stop=True); torch.cuda.synchronize()
    t0 = time.perf_counter(); c = P.simulate(g, s, s2, 1, 0, 1 << 17, 30, early_stop=True).cpu().tolist(); t = time.perf_counter() - t0
    print(f"simulate C4 ND {ebn0} dB 2^17 frames: {c[0] / t:.1f} frames/s incl. channel, mean it {c[4] / c[0]:.2f}, FER {c[2] / c[0]:.4f}")
PY
