"""B200-native implicit particle mover + moment interpolation.

A from-scratch sm_100a implementation of the data-parallel hot path of
sputniPIC (arXiv 2008.04397) as realised by the reference ``batchpic``
package: the fused implicit mover with trilinear E/B gather and the exact
int64 deposition of rho, J and the pressure tensor.  ``kernels`` is the
drop-in for ``batchpic.kernels``; ``mover`` mirrors ``batchpic.mover``;
``pipeline`` is the device-resident cycle driver (phases 1-3 and the
periodic sort of ``batchpic.pipeline.run_cycle``) with NCCL particle
decomposition and pinned-host batching.
"""

__version__ = "0.1.0"
