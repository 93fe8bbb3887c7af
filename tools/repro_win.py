import sys; sys.path.insert(0,'.')
import paper_1912_07423_b200 as synq
for model, n in (("pingpong", 0), ("brunel+", 400), ("vogels", 1000)):
    try:
        s = synq.Sim(model, n, synq.Opts(seed=42, deterministic=True, persistent=0, record=True))
        s.run(50); print(model, "ok", s.counters(), flush=True)
    except Exception as e:
        print(model, "ERR", e, flush=True)
