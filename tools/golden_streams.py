"""Write tests/golden/stream_sha256.json: sha256 of the input field and of
the ORACLE's stream (oracle.compress, single thread) for the full-size
configs cfg1-cfg4 (BASELINE.json configs[0..3]).  Calls only oracle/ and
synth/ — no CUDA path — so the stored hashes are expected values in the sense
of the parity rule (a stored value is written by a committed script that
calls only the oracle).  cfg3 takes ~6 min single-threaded."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth.fields import CONFIGS, eps_noa, sha256  # noqa: E402

out = {}
for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg4", "cfg3"]:
    cfg = CONFIGS[name]
    x = cfg.generate()
    eps = eps_noa(x, cfg.rel)
    t = time.time()
    st = oracle.compress(x, eps)
    out[name] = {"input_sha256": sha256(x), "eps": eps, "stream_bytes": len(st),
                 "stream_sha256": hashlib.sha256(st).hexdigest(), "oracle_s": round(time.time() - t, 1)}
    print(name, out[name], flush=True)
p = os.path.join(ROOT, "tests", "golden", "stream_sha256.json")
old = json.load(open(p)) if os.path.exists(p) else {}
old.update(out)
json.dump(old, open(p, "w"), indent=1, sort_keys=True)
