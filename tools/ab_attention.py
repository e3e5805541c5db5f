"""A/B: engine logits with the tcgen05 attention vs the mma.sync kernel (same trace)."""
import os, subprocess, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def run():
    import paper_2604_22881_b200 as mtkv
    kv = mtkv.KVConfig(num_layers=2, num_heads=2, head_dim=128, page_size=32, chunk_size=64, device_pages=256,
                       offload_quota=1024)
    m = mtkv.ModelConfig(num_layers=2, num_heads=2, head_dim=128, vocab=256, seed=3)
    rng = np.random.default_rng(0)
    eng = mtkv.Engine(kv, mode="hierarchical", backend="value", batch_size=4, model=m, keep_logits=True,
                      profile=True)
    out, ms = [], []
    for b in range(6):
        batch = [{"user": u, "tokens": rng.integers(0, 256, 300 if b == 0 else 40).tolist(),
                  "cands": rng.integers(0, 256, 8).tolist()} for u in range(4)]
        eng.process_batch(batch)
        out.append(eng.last_logits())
        ms.append(eng.last_attention_ms()[0])
    return np.concatenate(out), ms

if __name__ == "__main__":
    if len(sys.argv) > 1:
        lg, ms = run()
        np.save(sys.argv[1], lg)
        print(json.dumps({"attn_ms": ms}))
    else:
        a = subprocess.run([sys.executable, __file__, "/tmp/tc.npy"], capture_output=True, text=True)
        b = subprocess.run([sys.executable, __file__, "/tmp/mma.npy"], capture_output=True, text=True,
                           env={**os.environ, "MTKV_ATTN": "mma"})
        print("tc", a.stdout.strip(), a.stderr[-500:])
        print("mma", b.stdout.strip(), b.stderr[-500:])
        x, y = np.load("/tmp/tc.npy"), np.load("/tmp/mma.npy")
        rel = np.abs(x - y).max(1) / np.abs(y).max(1)
        print("tc vs mma logits: max rel diff", rel.max(), "identical:", np.array_equal(x, y))
