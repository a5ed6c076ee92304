"""Rebuild the DR specs of make_config_golden.py with the product's classes (tests)."""


def build(desc):
    from paper_2503_09203_b200.randomization import DRParameter, Gaussian, Piecewise, Uniform

    out = {}
    for key, d in desc.items():
        if d[0] == "uniform":
            dist = Uniform(d[1], d[2])
        elif d[0] == "gaussian":
            dist = Gaussian(d[1], d[2], (d[3], d[4]))
        else:
            dist = Piecewise(d[1], d[2])
        out[key] = DRParameter(key, dist)
    return out
