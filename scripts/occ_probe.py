import sys; sys.path.insert(0,'.')
from paper_2305_18057_b200 import inputs as I, sfv
X,Y=I.config_nodes("C2"); c=I.CONFIGS["C2"]
s=sfv.Solver(I.default_config(c["ni"],c["nj"]),X,Y)
print(sfv.LIB_PATH, s.launch_info())
