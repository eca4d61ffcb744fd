"""Debug: dump the slice partials (m, s, u, ya) of a V = 1 call."""
import torch, synth
from paper_2605_14220_b200 import tim
DEV = "cuda"
W = synth.head_weight(1, 128, 9, device=DEV)
ids = torch.zeros(8, dtype=torch.int64, device=DEV)
H = synth.hidden_states(8, 128, 9, device=DEV, weight=W, ids=ids, mode="flat")
lp, ent = tim.logprob(H, W, ids)
torch.cuda.synchronize()
ws = [v for k, v in tim._ws_cache.items() if k[2] == "logprob"][0]
part = ws[1024:1024 + 16 * 8].view(torch.float32).view(8, 4).cpu()
print("lp", lp.cpu().tolist())
print("ent", ent.cpu().tolist())
print("partials (m, s, u, ya):")
for r in part.tolist():
    print(["%.9g" % x for x in r])
