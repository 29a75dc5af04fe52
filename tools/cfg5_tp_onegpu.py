"""Config 5 (70B-shape target) with TP = 8 Megatron shards on ONE B200 through the in-process
TP group (8 rank threads on one device, rank-ordered device sums), against the unsharded TP = 1
engine on the same device: the full-size sharded path instantiated (8 x 17.6 GB target shards +
8 replicated 1B drafts ~ 161 GB), every rank's round results identical, and the committed tokens
equal to the unsharded engine's. A correctness run, not a timing: the 8 ranks share one GPU.
Usage: python tools/cfg5_tp_onegpu.py [tp]"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2604_20503_b200 import abi, engine, llama  # noqa: E402


def serve(eng, prompts, max_out, ks, out, idx):
    for i, (p, m) in enumerate(zip(prompts, max_out)):
        eng.submit(i, p, m)
    rounds, s = [], 0
    while eng.live_requests():
        live = eng.live_requests()
        eng.set_spec_lengths(live, [ks[(r + s) % len(ks)] for r in live])
        rounds.append([r.as_tuple() for r in eng.step()])
        s += 1
    out[idx] = ([eng.committed(i) for i in range(len(prompts))], rounds)


def make(desc, **kw):
    return engine.ServingEngine(desc=desc, max_batch=2, max_seq_len=128, mode=abi.MODE_VSD, default_spec_length=4,
                                max_spec_length=8, prefill_rows=256, **kw)


def main():
    tp = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    desc = llama.config5()
    V = desc.target.vocab
    rng = np.random.default_rng(5)
    prompts = [rng.integers(0, V - 1, size=40).tolist(), rng.integers(0, V - 1, size=23).tolist()]
    max_out = [12, 9]
    ks = [4, 2, 6]
    t0 = time.time()
    ref = [None]
    with make(desc) as e1:
        serve(e1, prompts, max_out, ks, ref, 0)
    t1 = time.time()
    group = engine.TpGroup.local(tp)
    engines = [make(desc, tp_size=tp, tp_rank=r, tp_group=group) for r in range(tp)]
    outs = [None] * tp
    th = [threading.Thread(target=serve, args=(engines[r], prompts, max_out, ks, outs, r)) for r in range(tp)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=1200)
    for e in engines:
        e.close()
    group.close()
    t2 = time.time()
    ok_ranks = all(o is not None for o in outs) and all(outs[r] == outs[0] for r in range(1, tp))
    same = outs[0] is not None and outs[0][0] == ref[0][0]
    print(json.dumps({"config": "cfg5 70B-shape target", "tp": tp, "ranks_identical": ok_ranks,
                      "tokens_equal_unsharded": same, "unsharded": ref[0][0], "sharded": outs[0][0] if outs[0] else None,
                      "rounds": len(ref[0][1]), "s_tp1": round(t1 - t0, 1), "s_tp": round(t2 - t1, 1)}), flush=True)
    return 0 if ok_ranks and same else 1


if __name__ == "__main__":
    sys.exit(main())
