// The opaque C-ABI handles of include/twg.h (shared by capi.cu and group.cu).
#pragma once

#include "walk.cuh"
#include "window.cuh"

struct twg_ctx {
  twg::Ctx c;
};
struct twg_store {
  twg::Store* s;
};
struct twg_window {
  twg::Window* w;
  twg_ctx* ctx;
};
struct twg_walkset {
  twg::WalkSetDev* w;
};

namespace twg {
// twg_last_error()'s message for this thread
void set_last_error(const char* what);
}  // namespace twg
