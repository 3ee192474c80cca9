"""dev: median group-seed and zeta wall times from DRZG_VERBOSE k3loop output (first two calls dropped)"""
import sys, re
L = sys.stdin.read().splitlines()
g = [float(x.split()[-1]) for x in L if "group seeds" in x][2:]
w = [float(x.split()[2]) for x in L if re.match(r"^\d+ wall ", x)][2:]
print("group seeds med", sorted(g)[len(g) // 2], "wall med", sorted(w)[len(w) // 2], "min", min(w))
