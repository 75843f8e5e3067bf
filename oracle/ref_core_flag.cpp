// TEST INFRASTRUCTURE ONLY. Linked beside the reference's own src/core.cpp: tells the tests that
// make_config in oracle/_ref/libbht_ref.so is the reference's code (see ref_core_min.cpp).
extern "C" __attribute__((visibility("default"))) int ref_core_is_reference() { return 1; }
