"""Operation tallies (counters.py:6-46 of the reference).

The device path increments these with exactly the reference's laws -- one
SpMV per operator application, 3 dots per CGS2 step, 2 per polynomial build
-- so cost reports and history rows are identical.  Pure host bookkeeping."""

from dataclasses import dataclass


@dataclass
class CostCounters:
    spmvs: int = 0
    dots: int = 0
    scalar_dots: int = 0
    vector_updates: int = 0
    prec_applies: int = 0

    def snapshot(self):
        return (self.spmvs, self.dots, self.scalar_dots, self.vector_updates,
                self.prec_applies)

    def as_dict(self):
        return {k: getattr(self, k) for k in
                ("spmvs", "dots", "scalar_dots", "vector_updates", "prec_applies")}
