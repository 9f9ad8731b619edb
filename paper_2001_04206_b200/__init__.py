"""paper_2001_04206_b200 -- B200-native (sm_100a) backpropagation of
Deep-Netts-style fully connected layers: the hot path arXiv 2001.04206
offloads (output error, hidden delta pass, weight/bias gradient outer
products, SGD/momentum update), behind the reference's ``lane`` layer/network
API.  See DESIGN.md; the C ABI is include/lane_b200.h; the Python mirror of
the reference API is :mod:`paper_2001_04206_b200.lane`.
"""

__all__ = ["lane"]


def __getattr__(name):
    if name == "lane":
        import importlib
        return importlib.import_module(".lane", __name__)
    raise AttributeError(name)
