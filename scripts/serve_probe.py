"""Where the serving clock goes (bench.py --serve [--tiered]): admit
(prefill) vs decode-step time, and the slow steps."""
import json
import sys
import types

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2511_00868_b200 import serving  # noqa: E402

rec = []
orig_init = serving.ServingLoop.__init__


def init(self, engine, *a, **k):
    orig_init(self, engine, *a, **k)
    eng = engine

    def timer(fn):
        kind = "step" if fn == eng.step else "admit"
        info = (len(getattr(eng, "_initial_rows", ())), len(getattr(eng, "_evict_pending", {}) or {}),
                eng.is_rerank_step())
        dt = self._time(fn)
        rec.append((kind, dt, info))
        return dt
    self.timer = timer


serving.ServingLoop.__init__ = init
args = types.SimpleNamespace(tiered="--tiered" in sys.argv)
bench.run_serve(args)
steps = [r for r in rec if r[0] == "step"]
admits = [r for r in rec if r[0] == "admit"]
slow = [r for r in steps if r[1] > 0.005]
out = {"admit_s": sum(r[1] for r in admits), "n_admit": len(admits),
       "step_s": sum(r[1] for r in steps), "n_step": len(steps),
       "slow_steps": len(slow), "slow_s": sum(r[1] for r in slow),
       "slow_with_initial": sum(1 for r in slow if r[2][0] > 0),
       "slow_rerank": sum(1 for r in slow if r[2][2]),
       "slow_sample": [(round(r[1] * 1e3, 2), r[2]) for r in slow[:12]],
       "admit_sample_ms": [round(r[1] * 1e3, 2) for r in admits[:12]]}
print(json.dumps(out))
