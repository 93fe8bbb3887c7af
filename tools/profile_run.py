"""Small driver for ncu captures: build a network through the C ABI and run
N steps in batches.  Usage: python tools/profile_run.py MODEL SYNAPSES STEPS BATCH"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_07423_b200 as synq

model, syn, steps, batch = sys.argv[1], float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
prof = os.environ.get('SYNQ_PROFILE') == '1'
sim = synq.Sim(model, opts=synq.Opts(seed=1, deterministic=True, batch_steps=batch, profile=prof), synapses=int(syn))
sim.run(steps)
c = sim.counters()
dev, ker = sim.device_time()
print(f"{model} syn={sim.synapses} n={sim.neurons} steps={steps} spikes={c['spikes']} "
      f"deliveries={c['deliveries']} device_s={dev:.4f} kernel_s={ker:.4f} "
      f"us/step={ker / steps * 1e6:.2f} launches={sim.kernel_launches()}")
if prof:
    pc = sim.phase_cycles()
    print('update detail (pacing):', pc.get('update_detail'))
    print('pipeline slots (cycles/step; passes per step):', pc.get('pipeline'))
    for key in ('mean', 'pacing'):
        tot = sum(pc[key].values())
        print(f'phase cycles/step ({key}, {pc["tiles"]} CTAs):', pc[key], 'total', round(tot),
              f'= {tot / 1.965e3:.2f} us at 1965 MHz')
