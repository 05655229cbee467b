"""Parameter shape catalogs of the benchmark workloads.

Mirrors catalogs.py:20-42 (ParamSpec: 1-d tensors are uncompressed biases,
higher-rank tensors compress as (shape[0], prod(shape[1:])) row-major views)
and the two built-in catalogs catalogs.py:65-109, in catalog order — the
order matters because `param_index` (biases included) seeds each Q.
"""

from dataclasses import dataclass
from math import prod

from .linalg import ContractViolation


@dataclass(frozen=True)
class ParamSpec:
    name: str
    shape: tuple

    def __post_init__(self):
        if len(self.shape) < 1 or any(d < 1 for d in self.shape):
            raise ContractViolation(f"bad shape for {self.name}: {self.shape}")

    @property
    def is_bias(self):
        return len(self.shape) == 1

    @property
    def size(self):
        return prod(self.shape)

    @property
    def matrix_shape(self):
        if self.is_bias:
            raise ContractViolation(f"{self.name} is a bias vector")
        return self.shape[0], prod(self.shape[1:])


@dataclass(frozen=True)
class ModelCatalog:
    name: str
    params: tuple


def _cat(name, rows):
    return ModelCatalog(name, tuple(ParamSpec(n, s) for n, s in rows))


RESNET18 = _cat("resnet18", [
    ("layer4.1.conv2", (512, 512, 3, 3)), ("layer4.0.conv2", (512, 512, 3, 3)),
    ("layer4.1.conv1", (512, 512, 3, 3)), ("layer4.0.conv1", (512, 256, 3, 3)),
    ("layer3.1.conv2", (256, 256, 3, 3)), ("layer3.1.conv1", (256, 256, 3, 3)),
    ("layer3.0.conv2", (256, 256, 3, 3)), ("layer3.0.conv1", (256, 128, 3, 3)),
    ("layer2.1.conv2", (128, 128, 3, 3)), ("layer2.1.conv1", (128, 128, 3, 3)),
    ("layer2.0.conv2", (128, 128, 3, 3)), ("layer4.0.shortcut.0", (512, 256, 1, 1)),
    ("layer2.0.conv1", (128, 64, 3, 3)), ("layer1.1.conv1", (64, 64, 3, 3)),
    ("layer1.1.conv2", (64, 64, 3, 3)), ("layer1.0.conv2", (64, 64, 3, 3)),
    ("layer1.0.conv1", (64, 64, 3, 3)), ("layer3.0.shortcut.0", (256, 128, 1, 1)),
    ("layer2.0.shortcut.0", (128, 64, 1, 1)), ("linear", (10, 512)),
    ("conv1", (64, 3, 3, 3)), ("bias_vectors", (9728,)),
])

LSTM = _cat("lstm", [
    ("encoder", (28869, 650)),
    ("rnn.ih.l0", (2600, 650)), ("rnn.hh.l0", (2600, 650)),
    ("rnn.ih.l1", (2600, 650)), ("rnn.hh.l1", (2600, 650)),
    ("rnn.ih.l2", (2600, 650)), ("rnn.hh.l2", (2600, 650)),
    ("bias_vectors", (44469,)),
])


def stress(n_mats=256, dim=4096):
    """BASELINE.json configs[4]: 256 matrices of 4096 x 4096, no bias."""
    return _cat(f"stress{n_mats}x{dim}", [(f"w{i}", (dim, dim)) for i in range(n_mats)])


BUILTIN = {"resnet18": RESNET18, "lstm": LSTM}


def get_catalog(name):
    if name in BUILTIN:
        return BUILTIN[name]
    if name.startswith("stress"):
        return stress()
    raise ContractViolation(f"unknown catalog {name!r}; choose from {sorted(BUILTIN)} or stress")
