"""paper_2404_01817_b200: B200-native (sm_100a) population-parallel NEAT.

Drop-in for the hot path of the reference ``arrayneat`` (TensorNEAT,
arXiv 2404.01817): the same function names, argument meaning and exceptions,
executed by hand-written CUDA kernels in the in-tree ``libtneat.so`` (C ABI,
include/tneat.h).  There is no CPU fallback.
"""

from .config import NeatConfig, dump_config, load_config, parse_config_text
from .errors import (ArrayNeatError, BadAttrIndex, CapacityFull, ConfigError, CycleDetected,
                     DanglingEndpoint, DuplicateConn, DuplicateKey, ExtinctionError,
                     IntegrityError, InvalidInput, KeyNotFound, ParseError, ProtectedNode,
                     ShapeMismatch, TerminalState)
from .functions import (ACTIVATION_IDS, AGGREGATION_IDS, DEFAULT_REGISTRY,
                        EXTENDED_AGGREGATION_IDS, FunctionRegistry)
from .genome import GenomeTensors, PopulationTensors
from .inference import (StackedNetworks, TransformedNetwork, finalize_transform, forward,
                        forward_arrays, forward_batch, forward_device, population_forward,
                        population_transform, transform, transform_arrays,
                        transform_population_stacked)

__version__ = "0.1.0"
