import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fstgen
import paper_2110_02848_b200 as p
V = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
A, _ = fstgen.config_c4(V=V, D=8)
Id = fstgen.identity_fst(range(16))
for X, Y, name in ((A, Id, "A o Id"), (Id, A, "Id o A")):
    c = p.compose(X, Y)
    print(name, c["num_states"], c["num_arcs"], flush=True)
