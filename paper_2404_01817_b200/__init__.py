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
from .genome import (ConnRow, GenomeTensors, NodeRow, PopulationTensors, count_live, genomes_equal,
                     init_arrays, init_genome)
from .inference import (StackedNetworks, TransformedNetwork, finalize_transform, forward,
                        forward_arrays, forward_batch, forward_device, population_forward,
                        population_transform, transform, transform_arrays,
                        transform_population_stacked)
from . import evolution, problems, rng  # noqa: E402  (module attributes)
from .evolution import (GenerationStats, NodeKeyAllocator, SpeciesState, allocate_spawns, crossover,
                        crossover_arrays, distance, distance_arrays, evolve_step, mutate, mutate_arrays,
                        reproduce, speciate, update_stagnation)
from .problems import (CartPoleProblem, CartPoleState, Problem, RegressionProblem, XorProblem,
                       cartpole_step, eval_cartpole, eval_regression, eval_xor, evaluate_population,
                       make_problem)
from .rng import RngStream
from .artifacts import check_integrity, parse_genome, serialize_genome
from .runner import (EvolutionState, RunOutcome, init_state, load_checkpoint, run_bench, run_experiment,
                     save_checkpoint)

__version__ = "0.1.0"
