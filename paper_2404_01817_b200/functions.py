"""Function code tables (reference functions.py:20-79).

On the GPU the activation/aggregation functions are compiled into the forward
kernels (csrc/common.cuh ``apply_act`` / ``agg_combine``), so the registry is a
code table only.  Codes follow the reference: activations 0 identity, 1 tanh,
2 sigmoid, 3 relu; aggregations 0 sum, 1 product, 2 max, 3 mean.  Code 4
(``min``) is an extension the north star asks for (no reference oracle).
Custom callables (reference ``FunctionRegistry(activations=...)``) cannot run
inside a CUDA kernel; passing a registry whose tables differ from the built-in
ones raises ``ConfigError`` instead of silently computing something else.
"""

from __future__ import annotations

import sys

from .errors import ConfigError

ACTIVATION_NAMES = {0: "identity", 1: "tanh", 2: "sigmoid", 3: "relu"}
AGGREGATION_NAMES = {0: "sum", 1: "product", 2: "max", 3: "mean", 4: "min"}
ACTIVATION_IDS = {v: k for k, v in ACTIVATION_NAMES.items()}
AGGREGATION_IDS = {v: k for k, v in AGGREGATION_NAMES.items() if k < 4}
EXTENDED_AGGREGATION_IDS = {v: k for k, v in AGGREGATION_NAMES.items()}


class FunctionRegistry:
    """Code table with the reference's lookup methods (functions.py:45-76)."""

    def __init__(self, activations: dict | None = None, aggregations: dict | None = None):
        self.activations = {k: (v, None) for k, v in ACTIVATION_NAMES.items()} \
            if activations is None else dict(activations)
        self.aggregations = {k: (v, None) for k, v in AGGREGATION_NAMES.items()} \
            if aggregations is None else dict(aggregations)

    def activation_id(self, name: str) -> int:
        for code, entry in self.activations.items():
            if (entry[0] if isinstance(entry, tuple) else entry) == name:
                return code
        raise ConfigError(f"unknown activation function {name!r}")

    def aggregation_id(self, name: str) -> int:
        for code, entry in self.aggregations.items():
            if (entry[0] if isinstance(entry, tuple) else entry) == name:
                return code
        raise ConfigError(f"unknown aggregation function {name!r}")

    def check_builtin(self) -> None:
        """The GPU kernels implement exactly the built-in code table."""
        for table, builtin, kind in ((self.activations, ACTIVATION_NAMES, "activation"),
                                     (self.aggregations, AGGREGATION_NAMES, "aggregation")):
            for code, entry in table.items():
                name = entry[0] if isinstance(entry, tuple) else entry
                if builtin.get(int(code)) != name:
                    raise ConfigError(
                        f"{kind} code {code} ({name!r}) is not a built-in GPU function; "
                        "custom functions are not supported on the device path")


DEFAULT_REGISTRY = FunctionRegistry()


def check_registry(registry) -> None:
    """Accept our registry, the reference's default registry, or None."""
    if registry is None or registry is DEFAULT_REGISTRY:
        return
    if isinstance(registry, FunctionRegistry):
        registry.check_builtin()
        return
    # a reference arrayneat.FunctionRegistry: compare names code by code, and
    # the callables against the built-in tables of the registry's own module
    # (a custom function registered under a built-in name is still custom)
    acts = getattr(registry, "activations", None)
    aggs = getattr(registry, "aggregations", None)
    if acts is None or aggs is None:
        raise ConfigError("registry must provide activations/aggregations tables")
    FunctionRegistry(acts, aggs).check_builtin()
    mod = sys.modules.get(type(registry).__module__)
    for table, base_name, kind in ((acts, "ACTIVATIONS", "activation"), (aggs, "AGGREGATIONS", "aggregation")):
        base = getattr(mod, base_name, None)
        if not isinstance(base, dict):
            continue
        for code, entry in table.items():
            fn = entry[1] if isinstance(entry, tuple) and len(entry) > 1 else None
            ref = base.get(int(code))
            if fn is not None and ref is not None and fn is not ref[1]:
                raise ConfigError(f"{kind} code {code} ({entry[0]!r}) is a custom callable; only the built-in "
                                  "functions are compiled into the device kernels")
