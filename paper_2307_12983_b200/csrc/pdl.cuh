// Programmatic dependent launch (PDL), device side.  Every kernel of the
// library starts with pdl::entry(): it waits until the preceding kernel on
// the stream has completed and its writes are visible (griddepcontrol.wait is
// a no-op for a normal launch), then lets the next kernel launch at once, so
// its CTAs are scheduled and run their prologue (barrier init, TMEM alloc,
// descriptor prefetch) while this grid drains.  Because every kernel waits
// before touching global memory, the chain keeps full stream order.
#pragma once

namespace pqlg::pdl {

__device__ __forceinline__ void wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void entry() {
  wait();
  trigger();
}

}  // namespace pqlg::pdl
