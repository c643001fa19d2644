import sys, json
sys.path.insert(0, '.')
import paper_2209_07632_b200 as vf
M = vf.ViewFactorMatrix.load('/tmp/cfg3.hvfm', 0)
print(json.dumps(M.refresh()))
