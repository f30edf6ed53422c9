"""Print the instruction-issue probes (integer roofline inputs)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2509_01654_b200 import _native
from paper_2509_01654_b200.engine import probe

res = {}
for name in _native.PROBES:
    ipc, ms = probe(name, 4000)
    res[name] = {"warp_instr_per_clk_per_sm": ipc, "ms": ms}
    print(f"{name:20s} ipc/SM={ipc:6.3f}  ms={ms:8.3f}")
print(json.dumps(res))
