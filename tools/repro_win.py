import sys; sys.path.insert(0,'.')
import numpy as np
import oracle
import paper_1912_07423_b200 as synq
n = 4000
s = synq.Sim("vogels", n, synq.Opts(seed=1, deterministic=True, record=True))
v0 = s.neuron_field(0).copy(); a0 = s.neuron_field(1).copy()
ref = oracle.Sim("vogels", n, 1)
s.run(1); ref.run(1)
v = s.neuron_field(0); rv = ref.field(0).view(np.float32)
for i in (0, 1, 1999, 2000, 2001, 2002, 3000, 3999):
    print(i, "init", v0[i], "acc0", a0[i], "gpu", v[i], "ref", rv[i], flush=True)
print("gpu==init for wrong:", int((v[2001:] == v0[2001:]).sum()))
idx = {float(x): k for k, x in enumerate(rv)}
print("gpu values found in ref at:", [idx.get(float(v[i])) for i in (2001, 2002, 2003, 3999)])
