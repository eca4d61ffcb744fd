"""Print the per-device SM -> die map the library probes (state 1 = valid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_14220_b200 import tim  # noqa: E402
import torch  # noqa: E402
st, die = tim.debug_die_map()
n = torch.cuda.get_device_properties(0).multi_processor_count
print("die map state", st, "die-1 SMs", sum(die[:n]), "".join(map(str, die[:n])))
