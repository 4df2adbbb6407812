"""Dev probe: graph-replayed steps vs eager steps (bitwise) and their timings."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
import oracle_lib
import paper_2009_09523_b200 as vnt

port = oracle_lib.port()
w = [784, 16, 10]
res = {}
for graphs in ("1", "0"):
    os.environ["VNT_GRAPHS"] = graphs
    e = vnt.Engine(w, "tanh", "softmax-cross-entropy", gemm_mode="ffma")
    e.add_device(1 << 20)
    e.set_params(port.init_params(w, 11))
    sizes, dev = vnt.uniform_mapping(256, 16, 1)
    losses = []
    for s in range(6):
        x, y = port.synth_batch(11, 60000, 784, 10, s * 256, 256)
        try:
            losses.append(e.train_step(x, y, sizes, dev, 0.05)[0])
        except Exception as ex:
            print("graphs", graphs, "step", s, "error", ex)
            raise
        print("graphs", graphs, "step", s, e.timings())
    res[graphs] = (e.get_params(), losses)
    e.close()
print("bitwise params", np.array_equal(res["1"][0], res["0"][0]), "losses", res["1"][1] == res["0"][1])
