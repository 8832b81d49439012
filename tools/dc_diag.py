import json, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2507_09730_b200.frwcap as frwcap
from paper_2507_09730_b200.workloads import c3_structure
from tests import scenes
from oracle.oracle import Oracle, Ref
doc = c3_structure(); text = json.dumps(doc); sc = scenes.scene_from_doc(doc)
from tests.test_gpu_transit_api import _free_points, _states
pts, hws = _free_points(sc, Ref().structure(sc), np.random.default_rng(3), 1)
c, h = [float(x) for x in pts[0]], float(hws[0])
eps, mask, tag, axis = frwcap.build_grid(text, c, h, 24)
st = _states(Oracle(), 5, 2000)
g = frwcap.transits_grid(eps, c, h, st)
np.save(sys.argv[1], np.stack([g["panel"], g["steps"], g["dir"]]))
print("distinct eps", len(np.unique(eps)))
