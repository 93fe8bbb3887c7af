"""Vogels 4000 on the persistent pipeline at several CTA counts (Opts(tiles)):
device ms per biological second after a 2000-step warm-up, state digest
(every tile count must agree bit for bit).
    python tools/vogels_tiles.py [TILES...]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq

for tiles in [int(x) or None for x in sys.argv[1:]] or [None, 8, 16, 24, 32, 48, 64]:
    sim = synq.Sim("vogels", 4000, synq.Opts(seed=1, deterministic=True, tiles=tiles))
    sim.run(2000)
    _, k0 = sim.device_time()
    sim.run(10000)
    _, k1 = sim.device_time()
    dig = hashlib.sha256(sim.neuron_field(0).tobytes()).hexdigest()[:12]
    print(f"tiles={tiles} engine={sim.engine}: {(k1 - k0) * 1e3:.2f} ms per bio-s, V {dig}", flush=True)
    sim.close()
