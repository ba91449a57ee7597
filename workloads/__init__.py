"""workloads -- seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

Holds only model parameter sets (as printed in the paper) and SDE simulators
(Euler--Maruyama data generation).  None of the method's arithmetic lives here.
"""
from .models import (LinearSpec, NonlinearSpec, wiener_velocity, ornstein_uhlenbeck,
                     coordinated_turn, van_der_pol, CONFIGS)
from .simulate import simulate_linear, simulate_nonlinear, make_workload

__all__ = ["LinearSpec", "NonlinearSpec", "wiener_velocity", "ornstein_uhlenbeck",
           "coordinated_turn", "van_der_pol", "CONFIGS", "simulate_linear",
           "simulate_nonlinear", "make_workload"]
