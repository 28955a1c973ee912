// Test stand-in naming the shipped program; the B200 path recognises the
// Dynamic driver and runs it natively (engine.compile_source).
Dynamic dynamicSSSP(Graph g) {}
