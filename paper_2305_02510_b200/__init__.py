"""B200-native engine for SuperNeuro's MAT-mode simulation step (and the
agent-based mode, ``abm_run``, on the same kernels).

The API mirrors the reference's ``spikeforge`` module (proj/python/spikeforge/
__init__.py) for the MAT path; compute runs in hand-written sm_100a kernels
behind the C ABI in ``include/superneuro_mat.h`` (``libsnmat.so``).
"""
from .model import (INFINITE_LEAK, NetworkDef, NeuronParams, RunResult, SimulationConfig,
                    SpikeEvent, SpikeRaster, StdpConfig, StimulusEntry, StimulusSchedule,
                    SynapseDef, WeightStorage, is_infinite_leak, leak_toward, raster_equal,
                    restrict_raster, validate_network, validate_stdp, validate_stimulus)
from .netgen import (BenchScenario, RandomStream, ScenarioBundle, SequentialRng, build_scenario,
                     erdos_renyi, mix64)
from .engine import MatEngine, comm_unique_id, device_count, partition_range, stdp_defaults
from .api import NeuromorphicModel, mat_run
from .abm import abm_run, behavior_names, register_stochastic_lif
from .lowering import LoweredNetwork, ProxyInfo, annotate_proxy_metadata, lower_delays, proxy_count
from .io import (FormatError, parse_network, parse_raster, parse_stdp, parse_stimulus,
                 serialize_network, serialize_stdp, write_raster, write_stimulus)

__all__ = [
    "INFINITE_LEAK", "NetworkDef", "NeuronParams", "RunResult", "SimulationConfig", "SpikeEvent",
    "SpikeRaster", "StdpConfig", "StimulusEntry", "StimulusSchedule", "SynapseDef",
    "WeightStorage", "is_infinite_leak", "leak_toward", "raster_equal", "restrict_raster",
    "validate_network", "validate_stdp", "validate_stimulus", "BenchScenario", "RandomStream",
    "ScenarioBundle", "SequentialRng", "build_scenario", "erdos_renyi", "mix64", "MatEngine",
    "comm_unique_id", "device_count", "partition_range", "stdp_defaults", "NeuromorphicModel",
    "mat_run", "abm_run", "behavior_names", "register_stochastic_lif", "LoweredNetwork",
    "ProxyInfo", "annotate_proxy_metadata", "lower_delays", "proxy_count", "FormatError", "parse_network", "parse_raster", "parse_stdp", "parse_stimulus",
    "serialize_network", "serialize_stdp", "write_raster", "write_stimulus",
]

__version__ = "0.1.0"
