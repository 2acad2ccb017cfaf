"""Golden fixtures for specdec.results_json: the REFERENCE's own report
(results_json, engine.cpp:531-587, via oracle/_ref's ref_decode) for C1-shaped
decodes, with the wall-clock fields dropped.  Run here, where /root/reference
is present:  python tests/golden/make_results_json.py"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle"))
import pyoracle as P  # noqa: E402

TIMING = ("prefill_seconds", "decode_seconds", "tokens_per_second_decode", "tokens_per_second_total")
CFG = dict(num_layers=2, num_heads=2, head_dim=8, vocab_size=259, max_positions=160, init_seed=0x10EA)


def main():
    ref = P.Reference()
    m = ref.model_init(CFG)
    for mname, mode in (("greedy", 0), ("vanilla", 1), ("ems", 2)):
        e = P.engine_config(mode=mode, predictor=1, k=4, copy_len=4, batch_size=3, max_new_tokens=24, seed=17,
                            stop_on_eos=1)
        js = ref.decode(e, m, P.CORPUS[:3])
        for k in TIMING:
            js["metrics"].pop(k)
        with open(os.path.join(HERE, f"results_json_retrieval_{mname}.json"), "w") as f:
            json.dump(dict(model=CFG, engine=e, prompts=P.CORPUS[:3], results=js), f, indent=1)
    ref.model_free(m)
    print("results_json fixtures written to", HERE)


if __name__ == "__main__":
    main()
