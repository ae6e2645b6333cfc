"""N4 measurement: dllm_lm_head_argmax at the LLaDA-8B LM-head shape (PAPER.md:516:
2,048 materialised-logit rows; d_model 4,096; vocab 126,464), CUDA events, L2
flushed between reps, one JSON line with the tensor roofline fraction."""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_17077_b200 import lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-tok", type=int, default=synth.LM_HEAD_FULL["n_tok"])
    ap.add_argument("--max-num-logits", type=int, default=synth.LM_HEAD_FULL["max_num_logits"])
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    f = synth.LM_HEAD_FULL
    n, d, v = args.n_tok, f["d_model"], f["vocab"]
    h, w = synth.lm_head_inputs(n, d, v, "realistic")
    h, w = h.cuda(), w.cuda()
    ids = torch.empty(n, dtype=torch.int32, device="cuda")
    ws = torch.empty(lib.lm_head_workspace_bytes(n, v, args.max_num_logits), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        lib.lm_head_argmax(h, w, ids, args.max_num_logits, ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        lib.lm_head_argmax(h, w, ids, args.max_num_logits, ws)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    t = statistics.median(ts)
    flop = 2.0 * n * d * v
    peak = 1642.7
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        pass
    print(json.dumps({"kernel": "dllm_lm_head_argmax", "shape": [n, d, v], "max_num_logits": args.max_num_logits,
                      "us_median": t * 1e6, "us_min": min(ts) * 1e6, "TFLOP/s": flop / t / 1e12,
                      "frac_of_bf16_peak": flop / t / 1e12 / peak, "peak": peak,
                      "weight_GB": v * d * 2 / 1e9, "logit_bytes_materialised": 0}))


if __name__ == "__main__":
    main()
