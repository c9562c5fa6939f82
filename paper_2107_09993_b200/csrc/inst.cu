// Per-dimensionality instances of the query pipeline (engine.cuh: Pipe).
// Compiled once per D with -DSKY_D=<D> (Makefile), so the 15 instances build
// in parallel instead of in one 3-minute translation unit.
#include "engine.cuh"

#ifndef SKY_D
#error "compile with -DSKY_D=<dimensionality>"
#endif

namespace skyeng {

template <int D>
void run_single_d(const Query& q, int kind) {
  if (kind == 0) {
    Pipe<float, float, true, D> p(q);
    p.run_single();
  } else if (kind == 1) {
    Pipe<float, double, false, D> p(q);
    p.run_single();
  } else {
    Pipe<double, double, false, D> p(q);
    p.run_single();
  }
}

template <int D>
void make_shard_d(const Query& q, int kind, std::unique_ptr<PipeBase>* out) {
  std::unique_ptr<PipeBase> p;
  if (kind == 0) p = std::make_unique<Pipe<float, float, true, D>>(q);
  else if (kind == 1) p = std::make_unique<Pipe<float, double, false, D>>(q);
  else p = std::make_unique<Pipe<double, double, false, D>>(q);
  p->local();
  *out = std::move(p);
}

template void run_single_d<SKY_D>(const Query&, int);
template void make_shard_d<SKY_D>(const Query&, int, std::unique_ptr<PipeBase>*);

}  // namespace skyeng
