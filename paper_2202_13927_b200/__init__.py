"""B200-native closed-loop Monte Carlo engine for virtual T1D trials.

Drop-in for the simulate / trial API of the reference ``glucotrial``
package (arXiv 2202.13927 hot path); compute runs in hand-written sm_100a
kernels behind the C-ABI in include/glucosim.h.
"""

from .analytics import (PatientStats, TrialAccumulator, build_trial_report, merge,
                        metric_quantiles, report_bytes)
from .config import SimulationConfig, SimulationError
from .controller import (ControllerHyperparameters, get_controller_factory, load_profile,
                         register_controller)
from .population import DevicePopulation, ParameterSet, Patient, generate_population
from .protocol import (Disturbance, FixedProtocol, Protocol, ThreeMealProtocol,
                       compile_protocol, validate_protocol)
from .simulation import (SimulationResult, SteadyStateError, TrialResult, run_trial,
                         simulate_closed_loop)
from .northern import NorthernYearProtocol
from .pid import PIDController, PIDProfile
from .population import validate_parameter_sets

__all__ = [
    "PatientStats", "TrialAccumulator", "build_trial_report", "merge", "metric_quantiles",
    "report_bytes", "SimulationConfig", "SimulationError", "ControllerHyperparameters",
    "get_controller_factory", "load_profile", "register_controller", "DevicePopulation",
    "ParameterSet", "Patient", "generate_population", "Disturbance", "FixedProtocol", "Protocol",
    "ThreeMealProtocol", "compile_protocol", "validate_protocol", "SimulationResult",
    "SteadyStateError", "TrialResult", "run_trial", "simulate_closed_loop", "NorthernYearProtocol",
    "PIDController", "PIDProfile", "validate_parameter_sets",
]
